# Quick GPU check: GPU tests, smoke, and an ncu launch list of smoke (the
# live dispatcher must complete under ncu's kernel serialisation).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke.txt 2>&1; echo "ncu smoke rc=$?"; tail -3 gpurun_out/ncu_smoke.txt; grep -c k_worker gpurun_out/launches_smoke.csv
