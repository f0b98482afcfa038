# Round 2 re-entry: state of the tree on the B200 — GPU tests, smoke, bench,
# config #3 variants.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
timeout 1200 python tools/hybrid_variants.py --horizon-ms 1000 --reps 3 --only A,B > gpurun_out/hybrid_variants.txt 2>&1; echo "hybrid rc=$?"; tail -4 gpurun_out/hybrid_variants.txt
