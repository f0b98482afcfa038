timeout 120 python tools/gemm_batch.py 200704 256 2304 3 2 1 1 2>&1 | tail -2
timeout 120 python tools/gemm_batch.py 200704 256 4608 3 2 1 1 2>&1 | tail -2
timeout 120 python tools/gemm_batch.py 200704 256 9216 3 2 1 1 2>&1 | tail -2
timeout 120 python tools/conv_batch.py 256 28 28 512 256 3 3 1 1 3 2>&1 | tail -2
timeout 120 python tools/conv_batch.py 256 28 28 1024 256 3 3 1 1 3 2>&1 | tail -2
