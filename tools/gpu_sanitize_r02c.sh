mkdir -p gpurun_out
export GPUOS_PIPELINE_TIMEOUT_MS=600000
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=k_worker --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.txt 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/sanitizer_$tool.txt
done
