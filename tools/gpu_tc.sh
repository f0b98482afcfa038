# Tensor-core bodies: parity tests + batch-mode throughput (conv / GEMM).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.txt
timeout 120 python tools/conv_batch.py 256 28 28 256 256 3 3 1 1 5 2>&1 | tail -3
timeout 120 python tools/conv_batch.py 256 14 14 512 512 3 3 1 1 3 2>&1 | tail -2
timeout 120 python tools/gemm_batch.py 8192 8192 8192 5 2 1 1 2>&1 | tail -3
timeout 120 python tools/gemm_batch.py 8192 8192 8192 3 2 32 1 2>&1 | tail -2
timeout 120 python tools/gemm_batch.py 2048 2048 2048 3 2 1 1 2>&1 | tail -2
