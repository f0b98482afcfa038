# Round 2 evidence pass: GPU tests, smoke, bench, ncu traffic of the
# saturation launches, ncu launch list of the bench, --set full of the conv
# body, sanitizers on smoke.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.txt
timeout 1500 python tools/ncu_traffic.py > gpurun_out/ncu_traffic.txt 2>&1; echo "ncu traffic rc=$?"; tail -4 gpurun_out/ncu_traffic.txt; cp profiles/ncu_traffic_r02.json gpurun_out/
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ncu_launches_bench.csv python bench.py --steps 2 --warmup 3 --skip-configs > gpurun_out/ncu_bench.txt 2>&1; echo "ncu launches rc=$?"; grep -c k_worker gpurun_out/ncu_launches_bench.csv
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_worker -c 1 -o gpurun_out/prof_conv_r02 python tools/sat_once.py conv > gpurun_out/ncu_conv_full.txt 2>&1; echo "ncu conv rc=$?"
export GPUOS_PIPELINE_TIMEOUT_MS=600000
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=k_worker --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_$tool.txt
done
