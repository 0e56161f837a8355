timeout 300 ncu --set full --import-source on -k regex:k_lrt5 -c 2 -o gpurun_out/lrt5 -f python tools/prof_lr.py C3 2 > gpurun_out/ncu_lrt5.log 2>&1
echo rc=$? >> gpurun_out/ncu_lrt5.log
tail -3 gpurun_out/ncu_lrt5.log
