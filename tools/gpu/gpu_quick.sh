# quick regression: Chebyshev/coverage/multirank tests + a short C3 bench (A/B against an env override)
timeout 900 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -p no:cacheprovider -rf -x > gpurun_out/quick.log 2>&1
echo "rc=$?" >> gpurun_out/quick.log; tail -4 gpurun_out/quick.log
for v in "" "SQNGD_LSPLIT=1"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded > gpurun_out/bench_q.log 2>&1
  python - "$v" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1])
print(sys.argv[1] or "default", 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'k_lrt us', round(d['roofline']['avg_launch_ms']*1e3,1), 'A', round(d['breakdown']['step_A_evals_per_s']), 'B', round(d['breakdown']['step_B_evals_per_s']))
PY
done
