set -x
for cfg in "--blocks-per-sm 4" "--blocks-per-sm 3" "--block 64 --blocks-per-sm 8" "--block 256 --blocks-per-sm 2" "--blocks-per-sm 5"; do
  timeout 300 python bench.py --steps 1 --warmup 3 --n-per-gpu 262144 --t-end 5 --no-cpu-baseline --no-e2e $cfg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['roofline']['kernel_ms'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
