mkdir -p gpurun_out
for v in x_a x_b x_c x_d; do
  echo "== $v" >> gpurun_out/exp.txt
  SG_LIB_PATH=paper_2104_05343_b200/libsg_$v.so timeout 120 python tools/flash_perf.py 32,512,16,64 >> gpurun_out/exp.txt 2>&1
  SG_LIB_PATH=paper_2104_05343_b200/libsg_$v.so timeout 120 python tools/ftrace.py bwd 2>&1 | head -8 >> gpurun_out/exp.txt
done
