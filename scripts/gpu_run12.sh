python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build12.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "config0 or config1_parity_ragged or hiv_short or hiv_full_horizon or invariance or shard or edge or numeric" > gpurun_out/pytest12.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest12.log
for g in keys=imm keys=param; do SSA_K1_GEN=$g timeout 300 python bench.py --steps 2 --warmup 2 --n-per-gpu 262144 --t-end 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('K1 $g', '%.4g ev/s' % d['value'], 'k1_ms=%.1f' % d['roofline']['kernel_ms'], 'frac=%.3f' % d['roofline']['frac'])"; done
timeout 600 python bench.py --steps 1 --warmup 1 --n-per-gpu 303104 --t-end 100 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('K1 N=303104 (4 full rounds)', '%.4g ev/s' % d['value'])"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:ssa_k2 -c 1 -o gpurun_out/k2_r1e python bench.py --config 3 --steps 1 --warmup 0 --n-per-gpu 65536 --t-end 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_k2e.log 2>&1; echo "ncu rc=$?"
