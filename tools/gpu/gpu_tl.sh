timeout 300 python tools/timeline.py C3 4 auto gpurun_out/timeline_c3.json > gpurun_out/timeline_c3.txt 2>&1
echo "timeline rc=$?"; grep -v "^  " gpurun_out/timeline_c3.txt | head -40
