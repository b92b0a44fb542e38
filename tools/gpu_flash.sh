mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_flash_gpu.py -x -q -p no:cacheprovider > gpurun_out/flash_test.log 2>&1; echo "rc $?" >> gpurun_out/flash_test.log
timeout 120 python tools/flash_perf.py 32,512,16,64 4,2048,16,64 > gpurun_out/flash_perf.txt 2>&1
SG_FTRACE_TIMELINE=20 timeout 120 python tools/ftrace.py bwd > gpurun_out/ftrace_bwd.txt 2>&1
