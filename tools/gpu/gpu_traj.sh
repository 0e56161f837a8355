# Alg. 1 trajectories on the final build (NEXT-3 PSL-vs-iteration): C1/C2 200, C3 500, C4 300 outer iterations,
# C2 with the ResNet generator; plus the stopping rule (patience 50) at C3
OUT=gpurun_out/traj.jsonl; rm -f $OUT
for a in "C1 200" "C2 200" "C3 500" "C4 300" "C2 200 0 1" "C3 2000 50"; do
  timeout 900 python tools/run_trajectory.py $a 2>/dev/null | tail -1 >> $OUT
done
python - <<'PY'
import json
for l in open('gpurun_out/traj.jsonl'):
    d=json.loads(l); print(d['config'], 'gen' if d['generator'] else '   ', d['engine'], 'T', d['T'], 'pat', d['patience'], 'it', d['iterations'], 'stopped', d['stopped'], f"start {d['start_pslr_db']:.2f} best {d['best_pslr_db']:.2f} dB @ {d['best_iter']}  device {d['device_s']:.2f} s")
PY
