mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_flash_gpu.py -x -q -p no:cacheprovider > gpurun_out/flash_test.log 2>&1; echo "rc $?" >> gpurun_out/flash_test.log
timeout 120 python tools/flash_perf.py 8,2048,32,128 4,2048,8,128 2,4096,32,128 > gpurun_out/flash_perf.txt 2>&1
echo "== v1" >> gpurun_out/flash_perf.txt
SG_FLASH_BWD128_V1=1 timeout 120 python tools/flash_perf.py 8,2048,32,128 4,2048,8,128 >> gpurun_out/flash_perf.txt 2>&1
