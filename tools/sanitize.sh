#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_probe.py), one
# tool at a time; logs under gpurun_out/sanitizer/.  Run under gpurun.
set -u
O=gpurun_out/sanitizer
mkdir -p $O
python tools/sanitize_probe.py > $O/plain.log 2>&1 || { echo "probe failed"; tail $O/plain.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 \
      python tools/sanitize_probe.py > $O/$tool.log 2>&1
  echo "$tool rc=$?: $(tail -1 $O/$tool.log)"
done

# compute-sanitizer is closed on this pool: the stand-in is the whole GPU suite
# on the debug-checks library (in-kernel bounds asserts + barrier jitter)
MSG_LIB_VARIANT=debug python -m pytest tests -m gpu -q --deselect tests/test_gpu_debug_build.py \
    > $O/pytest_gpu_debug_library.log 2>&1
echo "debug-library suite rc=$?: $(tail -1 $O/pytest_gpu_debug_library.log)"
