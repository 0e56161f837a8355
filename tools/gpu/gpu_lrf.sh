# k_lrf (tcgen05 forward) bring-up: a tiny forward first (hang guard), then the suites using the forward
timeout 120 python - <<'PY' > gpurun_out/lrf_smoke.log 2>&1
import numpy as np, torch
from paper_2604_25728_b200 import sqngd, inputs
from paper_2604_25728_b200.configs import Cfg
from oracle import oracle as O
c = Cfg("t", M=2, N=64, B=4, K=33, f_lo=-0.5, f_hi=0.5, R=1, r_n=4, doppler_engine=2)
z = inputs.phase_params(1, c.M, c.N, config_index=3); rho = inputs.init_thresholds(1, c.B, c.r_n)
q = O.quantize(c, z, rho); s = q["s_hard"]; w = s.astype(np.complex64)
ctx = sqngd.Context(c)
met, p, amap = ctx.af_forward(torch.as_tensor(s, device="cuda"), torch.as_tensor(w, device="cuda"), want_map=True)
m = ctx.metrics(met); ctx.sync()
ref, _, refmap = O.af(c, s, w, want_map=True) if 'want_map' in O.af.__code__.co_varnames else (O.af(c, s, w)[0], None, None)
print("gpu", m[0]["loss"], m[0]["wpsl"], "oracle", ref[0]["loss"], ref[0]["wpsl"])
print("engine", ctx.engine_info())
PY
echo "smoke rc=$?"; cat gpurun_out/lrf_smoke.log | tail -4
timeout 900 python -m pytest tests/test_gpu_chebyshev.py tests/test_gpu_coverage.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_parity.py tests/test_gpu_run.py -q -p no:cacheprovider -x > gpurun_out/lrf_tests.log 2>&1
echo "tests rc=$?"; tail -15 gpurun_out/lrf_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-torch --no-generator --batch-restarts 0 --no-work-sharded > gpurun_out/bench_q.log 2>&1
echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_q.log').read().strip().splitlines()[-1])
f=d['forward']
print('value', round(d['value']), 'e2e', round(d['e2e']['value']), 'MAX', round(d['breakdown']['max_mode_evals_per_s']), 'fwd cells/s %.3g' % f['cells_per_s'], 'fwd launch us', round(f['fused_launch_ms_no_map']*1e3,1), 'map frac', round(f['with_map']['roofline']['frac'],3), round(f['with_map']['roofline']['avg_launch_ms']*1e3,1), 'pitched', round(f['with_map_pitched']['roofline']['frac'],3), round(f['with_map_pitched']['roofline']['avg_launch_ms']*1e3,1))
PY
