mkdir -p gpurun_out
timeout 300 python tools/gemm_step_shapes.py > gpurun_out/gemm_step_shapes.txt 2>&1
timeout 300 python tools/gemm_ksweep.py > gpurun_out/gemm_ksweep.txt 2>&1
