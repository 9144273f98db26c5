#!/bin/bash
# compute-sanitizer's four tools over scripts/sanitize_case.py (logs and exit codes in gpurun_out/san_*)
rm -f gpurun_out/san_rc.txt
for t in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $t --error-exitcode 9 python scripts/sanitize_case.py > gpurun_out/san_$t.log 2>&1
  echo "$t rc=$?" >> gpurun_out/san_rc.txt
done
cat gpurun_out/san_rc.txt
