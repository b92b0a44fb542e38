# A/B the training step: this tree vs the copy under ab/old (built there), interleaved
for k in 1 2; do
  python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('new', round(d['value'],1), d['ms_per_step'], d['clocks']['sm_mhz'])"
  (cd ab/old && python bench.py --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('old', round(d['value'],1), d['ms_per_step'], d['clocks']['sm_mhz'])")
done
