# round-2 closing evidence: GPU tests, smoke, three bench lines, ncu launch list + GEMM traffic
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
for i in 1 2 3; do timeout 600 python bench.py > gpurun_out/bench_$i.json 2> gpurun_out/bench_$i.err; done
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r02c.csv python tools/one_step.py > gpurun_out/ncu1.log 2>&1
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:gemm_kernel --clock-control none --csv --log-file gpurun_out/gemm_traffic_r02c.csv python tools/one_step.py > gpurun_out/ncu2.log 2>&1
