#!/bin/bash
# compute-sanitizer pass over one prepared Newton step of each scene (memcheck
# with leak check, racecheck, synccheck) and the self-contact stencil tests
# (memcheck).  Outputs under gpurun_out/sanitize_*.log; summary on stdout.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for sc in ${@:-c1 c2 c3}; do
  for tool in memcheck racecheck synccheck; do
    extra=""; [ $tool = memcheck ] && extra="--leak-check full"
    timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 20 python tools/one_step.py $sc 1 \
      > gpurun_out/sanitize_${tool}_$sc.log 2>&1
    echo "$sc $tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_${tool}_$sc.log | tr '\n' ' ')"
  done
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q -m gpu \
  tests/test_contact4.py tests/test_self_contact.py > gpurun_out/sanitize_memcheck_contact.log 2>&1
echo "contact tests memcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/sanitize_memcheck_contact.log | tail -2 | tr '\n' ' ')"
