# round-2 evidence: C3 step launch list (cold-cache, serialised: compare shares) and ncu --set full of k_lrt
python tools/step_loop.py C3 3 > gpurun_out/sl_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_step_c3.csv python tools/step_loop.py C3 3 > gpurun_out/ncu_ll.log 2>&1
echo "ll rc=$?"
python tools/prof_lr.py C3 2 > gpurun_out/pl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_lrt -s 2 -c 2 -o gpurun_out/r02_lrt -f python tools/prof_lr.py C3 2 > gpurun_out/ncu_lrt.log 2>&1
echo "lrt rc=$?"
python tools/step_loop.py C3 2 fft > gpurun_out/sl_fft_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_af -s 6 -c 2 -o gpurun_out/r02_kaf -f python tools/step_loop.py C3 2 fft > gpurun_out/ncu_kaf.log 2>&1
echo "kaf rc=$?"
