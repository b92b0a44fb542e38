mkdir -p gpurun_out
for r in 1 2; do for d in 1 0; do
  echo "== die $d" >> gpurun_out/die_ab.txt
  SG_GEMM_DIE=$d timeout 300 python tools/gemm_group_sweep.py 16 >> gpurun_out/die_ab.txt 2>&1
done; done
