# GEMV pair runs: GEMV/chain/model GPU tests, batch GEMV rates, config #3 breakdown.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "gemv or chain or models or smoke" > gpurun_out/pytest_gemv.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gemv.txt
for shp in "4096 4096 3 32 8" "6144 4096 3 32 6" "262144 8192 3 32 1"; do timeout 120 python tools/gemv_batch.py $shp 2>&1 | tail -2; done
for sp in 6,8,1,9 3,4,1,4; do echo "== splits $sp"; timeout 300 python tools/hybrid_breakdown.py --train-alone --splits $sp 2>&1 | tail -15; done
