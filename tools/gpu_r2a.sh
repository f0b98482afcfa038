# Round 2: live breakdown, ncu of the live (ring-fed) fig7 run, sanitizers on
# the single-launch dispatcher, and the bench.
mkdir -p gpurun_out
bash tools/gpu_live_ncu.sh
export GPUOS_PIPELINE_TIMEOUT_MS=600000
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=k_worker --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.txt
done
unset GPUOS_PIPELINE_TIMEOUT_MS
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
