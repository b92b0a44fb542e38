mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do timeout 600 python -m pytest tests/test_dist.py -m gpu -q -p no:cacheprovider -k "graph and 2-4" 2>&1 | grep -E "^E  |passed|failed" | head -4 >> gpurun_out/dist_rep.log; done
