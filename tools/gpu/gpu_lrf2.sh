timeout 300 python tools/lrf_check.py > gpurun_out/lrf_check.log 2>&1; echo "check rc=$?"; tail -6 gpurun_out/lrf_check.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded > gpurun_out/bench_q.log 2>&1
echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1])
f=d['forward']
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'MAX', round(d['breakdown']['max_mode_evals_per_s']), 'fwd cells/s %.3g' % f['cells_per_s'], 'fwd launch us', round(f['fused_launch_ms_no_map']*1e3,1), 'map frac', round(f['with_map']['roofline']['frac'],3), round(f['with_map']['roofline']['avg_launch_ms']*1e3,1), 'pitched', round(f['with_map_pitched']['roofline']['frac'],3), round(f['with_map_pitched']['roofline']['avg_launch_ms']*1e3,1))
PY
