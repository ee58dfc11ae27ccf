mkdir -p gpurun_out
for p in 3 0 1; do SVB_GEMM_TRACE=1 timeout 200 python tools/gemm_trace.py $p >> gpurun_out/gemm_trace.txt 2>&1; done
SVB_GEMM_TRACE=1 SVB_GEMM_DEBUG=1 timeout 200 python tools/gemm_trace.py 3 >> gpurun_out/gemm_trace.txt 2>&1
