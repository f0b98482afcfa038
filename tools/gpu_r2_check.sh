# Quick check: model/decode GPU tests (tenant bodies in the decode trace),
# racecheck on smoke, decode breakdown, config #3 variant A.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "models or user_bodies or chain or scheduler" > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.txt
export GPUOS_PIPELINE_TIMEOUT_MS=600000
timeout 900 compute-sanitizer --tool racecheck --kernel-name kns=k_worker --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/sanitizer_racecheck.txt
unset GPUOS_PIPELINE_TIMEOUT_MS
timeout 300 python tools/hybrid_breakdown.py > gpurun_out/hb.txt 2>&1; head -3 gpurun_out/hb.txt | cut -c1-300
timeout 120 python tools/gemm_batch.py 8192 8192 8192 3 2 1 1 2>&1 | tail -2
