# full GPU suite (+ parity record) and smoke
SQNGD_PARITY_LOG=gpurun_out/parity_full.json timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/full.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
