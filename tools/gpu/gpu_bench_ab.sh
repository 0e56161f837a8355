# A/B: tcgen05 k_lrt5 (default) vs mma.sync k_lrt at C3 and C5, plus the timed forward
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 > gpurun_out/bench_tc5.log 2>&1
SQNGD_LR_TC5=0 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 > gpurun_out/bench_tc0.log 2>&1
timeout 600 python bench.py --config C5 --steps 2 --warmup 1 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 > gpurun_out/bench_tc5_c5.log 2>&1
for f in gpurun_out/bench_tc5.log gpurun_out/bench_tc0.log gpurun_out/bench_tc5_c5.log; do
python - "$f" <<'PY'
import json,sys
t=open(sys.argv[1]).read().strip().splitlines()
try:
  d=json.loads(t[-1])
  r=d['roofline']
  print(sys.argv[1], 'value', round(d['value']), 'e2e', round(d['e2e']['value']), 'kernel', r['kernel'], 'ms', round(r['avg_launch_ms']*1e3,1), 'us frac', round(r['frac'],3), 'tensor', round(r.get('pipes',{}).get('tensor',{}).get('frac',0),3), 'fwd cells/s %.3g'%d['forward']['cells_per_s'], 'map hbm frac', round(d['forward']['with_map']['roofline']['frac'],3), d['kernel_ms'])
except Exception as e:
  print(sys.argv[1], 'ERR', e, t[-5:])
PY
done
