# racecheck re-run after the two race fixes + per-phase cycle shares (c2, c4)
mkdir -p gpurun_out/r2b
CS=/usr/local/cuda/bin/compute-sanitizer
for spec in "c2 --graphs 48" "c3small --queries 16 --graphs 400" "c4 --graphs 3"; do
  set -- $spec
  timeout 900 $CS --tool racecheck --error-exitcode 99 --print-limit 20 python tools/sanitize_run.py $spec > gpurun_out/r2b/racecheck_$1.log 2>&1
  echo "racecheck $spec rc=$? :: $(grep -E 'RACECHECK SUMMARY|bitwise' gpurun_out/r2b/racecheck_$1.log | tr '\n' ' ')" >> gpurun_out/r2b/summary.txt
done
CFGSIM_PHASES=1 timeout 600 python tools/phases.py c2 > gpurun_out/r2b/phases_c2.txt 2>&1
CFGSIM_PHASES=1 timeout 600 python tools/phases.py c4 --graphs 60 > gpurun_out/r2b/phases_c4.txt 2>&1
