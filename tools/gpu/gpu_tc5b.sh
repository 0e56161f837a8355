export SQNGD_PARITY_LOG=gpurun_out/parity_tc5b.json
timeout 120 python -m pytest tests/test_gpu_chebyshev.py -q -x -p no:cacheprovider -k "forward_map_and_metrics and C1" > gpurun_out/tc5b_a.log 2>&1
echo "rc=$?" >> gpurun_out/tc5b_a.log; tail -2 gpurun_out/tc5b_a.log
timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 > gpurun_out/bench_tc5b.log 2>&1
python - gpurun_out/bench_tc5b.log <<'PY'
import json,sys
t=open(sys.argv[1]).read().strip().splitlines()
try:
  d=json.loads(t[-1]); r=d['roofline']
  print('value', round(d['value']), 'e2e', round(d['e2e']['value']), r['kernel'], 'us', round(r['avg_launch_ms']*1e3,1), 'frac', round(r['frac'],3), 'fwd cells/s %.3g'%d['forward']['cells_per_s'], d['kernel_ms'])
except Exception as e: print('ERR', e, t[-5:])
PY
timeout 600 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_coverage.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -rf > gpurun_out/tc5b_b.log 2>&1
echo "rc=$?" >> gpurun_out/tc5b_b.log; tail -8 gpurun_out/tc5b_b.log
timeout 300 ncu --set full --import-source on -k regex:k_lrt5 -c 2 -o gpurun_out/lrt5b -f python tools/prof_lr.py C3 2 > gpurun_out/ncu_lrt5b.log 2>&1
