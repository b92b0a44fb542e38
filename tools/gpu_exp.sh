mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_flash_gpu.py -x -q -p no:cacheprovider > gpurun_out/flash_test.log 2>&1; echo "rc $?" >> gpurun_out/flash_test.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 120 python tools/flash_perf.py > gpurun_out/flash_perf.txt 2>&1
timeout 900 python bench.py --workload gpt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gpt_train.json 2> gpurun_out/gpt_train.err
