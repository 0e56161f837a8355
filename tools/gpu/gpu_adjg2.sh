timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "clustered or chain" > gpurun_out/rhoclu.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/rhoclu.log
python tools/step_loop.py C3 2 > gpurun_out/sl_plain.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on \
  -k "regex:^(k_adj_g|k_node|k_grad_rho|k_adj_gc)$" -s 40 -c 8 -o gpurun_out/r02h_tails -f python tools/step_loop.py C3 2 > gpurun_out/ncu_tails.log 2>&1
echo "ncu rc=$?"
