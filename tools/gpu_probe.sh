mkdir -p gpurun_out
./tools/micro/mufu_mix > gpurun_out/mufu_mix.txt 2>&1
./tools/micro/umma_rate > gpurun_out/umma_rate.txt 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:flash_bwd2 -c 1 -o gpurun_out/flash_bwd64 -f python tools/flash_one.py 32 512 16 64 > gpurun_out/ncu_fb.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:gemm_kernel -c 1 -o gpurun_out/gemm_fc1 -f python tools/gemm_one.py fc1 1 > gpurun_out/ncu_fc1.log 2>&1
