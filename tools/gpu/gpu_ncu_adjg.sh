# ncu --set full of k_adj_g / k_node / k_rows_adam_w / k_combine_rows at C3 (pipeline cache state) + device timeline
python tools/step_loop.py C3 2 > gpurun_out/sl_plain.log 2>&1 && \
ncu --set full --clock-control none --cache-control none --import-source on \
  -k "regex:k_adj_g<|k_node|k_rows_adam_w|k_combine_rows" \
  -s 40 -c 4 -o gpurun_out/r02h_adjg -f python tools/step_loop.py C3 2 > gpurun_out/ncu_adjg.log 2>&1
echo "ncu rc=$?"
timeout 300 python tools/timeline.py C3 3 auto gpurun_out/timeline_c3.json > gpurun_out/timeline_c3.txt 2>&1; echo "tl rc=$?"
