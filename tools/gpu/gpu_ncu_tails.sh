# ncu --set full of the C3 step's tail kernels (one launch each, pipeline cache state)
python tools/step_loop.py C3 2 > gpurun_out/sl_plain.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on \
  -k "regex:k_adj_g|k_node|k_grad_rho_part|k_rows_adam_w|k_combine_rows|k_lr_finish|k_quantize|k_xhat|k_adam_project_rho" \
  -s 200 -c 12 -o gpurun_out/r02_tails -f python tools/step_loop.py C3 2 > gpurun_out/ncu_tails.log 2>&1
echo "tails rc=$?"
