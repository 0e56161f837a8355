# A/B of env settings / library variants on one box: short C3 bench per arm, alternated twice.
# AB_ARMS="default SQNGD_LRT_BAL=0 lib:nodepk"
for pass in 1 2; do
for v in $AB_ARMS; do
  lib=""; envs=""
  for part in ${v//,/ }; do
    case "$part" in lib:*) lib=tools/variants/libsqngd_${part#lib:}.so;; default) ;; *) envs="$envs $part";; esac
  done
  env $envs SQNGD_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded > gpurun_out/bench_ab.log 2>&1
  python - "$v" <<'PY'
import json,sys
try:
    d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
    print(f"{sys.argv[1]:18s} value {d['value']:.0f} ms/step {d['ms_per_step']:.4f} k_lrt {d['roofline']['avg_launch_ms']*1e3:.1f} us  A {d['breakdown']['step_A_evals_per_s']:.0f} B {d['breakdown']['step_B_evals_per_s']:.0f} fwd_nomap {d['forward']['fused_launch_ms_no_map']*1e3:.1f} us fft {d.get('fft_engine',{}).get('value',0):.0f}")
except Exception as e:
    print(sys.argv[1], "FAILED", e); print(open('gpurun_out/bench_ab.log').read()[-1500:])
PY
done; done
