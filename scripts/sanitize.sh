#!/bin/bash
# compute-sanitizer over every kernel family (run on the B200 box from the repo root).
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 \
    python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
