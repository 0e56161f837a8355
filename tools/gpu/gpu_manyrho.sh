for v in "" nocp; do
  lib=""; [ -n "$v" ] && lib=tools/variants/libsqngd_$v.so
  rm -f gpurun_out/mr_$v.json
  SQNGD_LIB=$lib SQNGD_PARITY_LOG=gpurun_out/mr_${v:-default}.json timeout 600 python -m pytest tests/test_gpu_coverage.py -q -p no:cacheprovider -k "many_thresholds" > /dev/null 2>&1
  python -c "
import json,sys; r=json.load(open('gpurun_out/mr_${v:-default}.json'))
for x in r: print('${v:-default}', x['test'][-40:], x['quantity'], '%.3g' % x['achieved'])"
done
