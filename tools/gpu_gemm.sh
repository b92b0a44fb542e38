mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_summa_gpu.py -x -q -p no:cacheprovider > gpurun_out/gemm_test.log 2>&1; echo "rc $?" >> gpurun_out/gemm_test.log
timeout 300 python tools/gemm_step_shapes.py > gpurun_out/gemm_step_shapes.txt 2>&1
for c in dmid fc1 dmidg dense; do echo "== $c"; python tools/gtrace.py $c; done > gpurun_out/gtrace.txt 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
