mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for pr in 256 128 0; do
  for g in 16 8; do
    echo "== promo $pr group $g" >> gpurun_out/big_exp.txt
    SG_TMA_L2_PROMOTION=$pr SG_GEMM_GROUP_M=$g timeout 300 $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:gemm_kernel -c 1 python tools/gemm_one_big.py 16384 sg 2>&1 | grep -E "duration|dram__bytes|hit_rate" >> gpurun_out/big_exp.txt
  done
done
