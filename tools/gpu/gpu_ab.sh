# A/B of library variants on one box: bench C3 (short) with SQNGD_LIB pointing at each variant
for v in "" $AB_VARIANTS "" $AB_VARIANTS; do
  lib=""; [ -n "$v" ] && lib=tools/variants/libsqngd_$v.so
  SQNGD_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded > gpurun_out/bench_ab.log 2>&1
  python - "${v:-default}" <<'PY'
import json,sys
d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1])
print(f"{sys.argv[1]:12s} value {d['value']:.0f} ms/step {d['ms_per_step']:.4f} k_lrt {d['roofline']['avg_launch_ms']*1e3:.1f} us  A {d['breakdown']['step_A_evals_per_s']:.0f} B {d['breakdown']['step_B_evals_per_s']:.0f} fwd_nomap {d['forward']['fused_launch_ms_no_map']*1e3:.1f} us fft {d.get('fft_engine',{}).get('value',0):.0f}")
PY
done
