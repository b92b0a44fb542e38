mkdir -p gpurun_out
timeout 120 python tools/flash_perf.py > gpurun_out/flash_perf.txt 2>&1
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:flash_bwd2 -c 1 -o gpurun_out/fb64_r02c -f python tools/flash_one.py 32 512 16 64 > gpurun_out/ncu_a.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:flash_bwd3 -c 1 -o gpurun_out/fb128_r02c -f python tools/flash_one.py 8 2048 32 128 > gpurun_out/ncu_b.log 2>&1
timeout 600 $NCU --set full --import-source on --clock-control none -k regex:flash_fwd2 -c 1 -o gpurun_out/ff128_r02c -f python tools/flash_one.py 8 2048 32 128 > gpurun_out/ncu_c.log 2>&1
