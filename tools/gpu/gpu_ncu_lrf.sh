python tools/prof_lr.py C3 2 > gpurun_out/pl_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_lrf" -s 1 -c 1 -o gpurun_out/r02_lrf -f python tools/prof_lr.py C3 2 > gpurun_out/ncu_lrf.log 2>&1
echo "lrf rc=$?"
