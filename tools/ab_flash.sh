# A/B: current libsg.so vs paper_2104_05343_b200/libsg_ab.so, interleaved
for k in 1 2 3; do
  echo "new"; python tools/flash_perf.py | grep -E "fwd|bwd"
  echo "old"; SG_LIB_PATH=paper_2104_05343_b200/libsg_ab.so python tools/flash_perf.py | grep -E "fwd|bwd"
done
