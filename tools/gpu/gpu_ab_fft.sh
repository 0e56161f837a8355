# A/B of library variants for the per-bin FFT engine: C3 (engine forced) and C4 step times
for v in "" $AB_VARIANTS "" $AB_VARIANTS; do
  lib=""; [ -n "$v" ] && lib=tools/variants/libsqngd_$v.so
  a=$(SQNGD_LIB=$lib timeout 300 python tools/step_loop.py C3 5 fft 2>&1 | tail -1)
  b=$(SQNGD_LIB=$lib timeout 300 python tools/step_loop.py C4 3 2>&1 | tail -1)
  echo "${v:-default}: $a | $b"
done
