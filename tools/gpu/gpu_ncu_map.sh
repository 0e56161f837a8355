# ncu --set full of the map-writing forward contraction (k_lrt mode 2) at C3
python tools/prof_lr.py C3 2 map > gpurun_out/pl_map_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_lrtILi10ELi1ELb0ELi2E" --kernel-name-base mangled -s 1 -c 1 -o gpurun_out/r02_lrt_map -f python tools/prof_lr.py C3 2 map > gpurun_out/ncu_map.log 2>&1
echo "map rc=$?"
