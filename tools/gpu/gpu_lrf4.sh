timeout 300 python tools/lrf_check.py > gpurun_out/lrf_check.log 2>&1; echo "check rc=$?"; tail -5 gpurun_out/lrf_check.log
timeout 600 python -m pytest tests/test_gpu_coverage.py tests/test_gpu_chebyshev.py -q -p no:cacheprovider -x -k "map or tcgen05 or forward" > gpurun_out/lrf_t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/lrf_t.log
for v in 1 2; do
SQNGD_LRF=$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded > gpurun_out/bench_q.log 2>&1
python - $v <<'PY'
import json,sys
d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1])
f=d['forward']
print('LRF', sys.argv[1], 'value', round(d['value']), 'MAX', round(d['breakdown']['max_mode_evals_per_s']), 'fwd launch us', round(f['fused_launch_ms_no_map']*1e3,1), 'map', round(f['with_map']['roofline']['frac'],3), round(f['with_map']['roofline']['avg_launch_ms']*1e3,1), 'pitched', round(f['with_map_pitched']['roofline']['frac'],3), round(f['with_map_pitched']['roofline']['avg_launch_ms']*1e3,1))
PY
done
