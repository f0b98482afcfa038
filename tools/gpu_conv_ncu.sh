# Conv body: batch throughput (1 and 32 atoms) and one ncu --set full capture.
mkdir -p gpurun_out
timeout 120 python tools/conv_batch.py 256 28 28 256 256 3 3 1 1 4 1 2>&1 | tail -2
timeout 120 python tools/conv_batch.py 256 28 28 256 256 3 3 1 1 4 32 2>&1 | tail -2
timeout 120 python tools/gemm_batch.py 8192 8192 8192 3 2 1 1 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_worker -c 1 -o gpurun_out/prof_conv python tools/conv_batch.py 256 28 28 256 256 3 3 1 1 1 1 > gpurun_out/ncu_conv.txt 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ncu_conv.txt
