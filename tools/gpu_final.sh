# end-of-session validation: GPU tests, smoke, two bench lines, GPT lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
for i in 1 2; do timeout 600 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; done
timeout 900 python bench.py --workload gpt --mode infer --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/gpt_infer.json 2> gpurun_out/gpt_infer.err
