#!/bin/bash
# compute-sanitizer sweep over reduced benchmark paths:
# memcheck / racecheck / synccheck on c2 (two-stage all-pairs), c3 and c3small
# (query-vs-corpus rectangles after a stage-2 launch), c4 (large-N kernel).
# Logs: gpurun_out/sanitize/<tool>_<config>.log; summary on stdout.
set -u
cd "$(dirname "$0")/.."
out=gpurun_out/sanitize
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool config args...
  local tool=$1 cfg=$2; shift 2
  local log="$out/${tool}_${cfg}.log"
  local t0=$(date +%s)
  timeout 1500 $CS --tool "$tool" --error-exitcode 99 --print-limit 50 python tools/sanitize_run.py "$cfg" "$@" > "$log" 2>&1
  local rc=$?
  local t1=$(date +%s)
  echo "$tool $cfg $* rc=$rc $((t1 - t0))s :: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|bitwise' "$log" | tr '\n' ' ')"
}
run memcheck c2 --graphs 160
run memcheck c3small --queries 100 --graphs 8000
run memcheck c3 --queries 100 --graphs 8000
run memcheck c4 --graphs 6
run racecheck c2 --graphs 48
run racecheck c3small --queries 16 --graphs 400
run racecheck c4 --graphs 3
run synccheck c2 --graphs 96
run synccheck c3small --queries 32 --graphs 1000
run synccheck c4 --graphs 4
