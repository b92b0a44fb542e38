mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 900 python bench.py --workload gpt --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/gpt_train.json 2> gpurun_out/gpt_train.err
timeout 900 python bench.py --workload gpt --mode infer --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gpt_infer.json 2> gpurun_out/gpt_infer.err
