# compute-sanitizer probe (one tool per call): is the tool usable on this box?
which compute-sanitizer; compute-sanitizer --version 2>&1 | head -3
timeout 900 compute-sanitizer --tool ${TOOL:-memcheck} --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/sanitize_${TOOL:-memcheck}.log 2>&1
echo "rc=$?"; tail -15 gpurun_out/sanitize_${TOOL:-memcheck}.log
