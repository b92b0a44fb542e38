# round-2 evidence set: GPU tests, bench line, ncu launch list of one step, GEMM traffic, flash --set full
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_r02b.csv python tools/one_step.py > gpurun_out/ncu1.log 2>&1
timeout 900 $NCU --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:gemm_kernel --clock-control none --csv --log-file gpurun_out/gemm_traffic_r02b.csv python tools/one_step.py > gpurun_out/ncu2.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:flash_bwd2 -c 1 -o gpurun_out/flash_bwd64_r02b -f python tools/flash_one.py 32 512 16 64 > gpurun_out/ncu3.log 2>&1
