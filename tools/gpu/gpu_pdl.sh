timeout 900 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_coverage.py tests/test_gpu_multirank.py tests/test_gpu_parity.py tests/test_gpu_status.py tests/test_gpu_run.py -q -p no:cacheprovider -x > gpurun_out/pdl_tests.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/pdl_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded > gpurun_out/bench_q.log 2>&1
echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1])
print('value', round(d['value']), 'ms/step', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['value']), 'k_lrt us', round(d['roofline']['avg_launch_ms']*1e3,1), 'A', round(d['breakdown']['step_A_evals_per_s']), 'B', round(d['breakdown']['step_B_evals_per_s']))
PY
timeout 300 python tools/timeline.py C3 3 auto gpurun_out/timeline_c3.json > gpurun_out/timeline_c3.txt 2>&1; sed -n 3,24p gpurun_out/timeline_c3.txt
