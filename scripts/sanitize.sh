#!/bin/bash
# Memory-safety checks of every kernel family (run on the B200 box from the repo root).
# compute-sanitizer is closed on the GPU pool (the harness refuses it: runs under it have left GPUs
# needing a reset), so the stand-in is the library's own device bounds checks (SSA_DEBUG_CHECKS=1:
# every index the event loops derive from model tables or trajectory state is range-checked and a
# violation fails the call) over small invocations of every kernel family and the GPU parity suite.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
SSA_DEBUG_CHECKS=1 timeout 900 python scripts/sanitize_run.py > gpurun_out/debugchecks_run.log 2>&1
echo "debug-checks kernel families rc=$? $(tail -1 gpurun_out/debugchecks_run.log)"
SSA_DEBUG_CHECKS=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_union.py \
  -q -m gpu > gpurun_out/debugchecks_pytest.log 2>&1
echo "debug-checks GPU parity suite rc=$? $(tail -1 gpurun_out/debugchecks_pytest.log)"
