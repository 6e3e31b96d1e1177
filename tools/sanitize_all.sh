#!/bin/bash
# compute-sanitizer sweep over small hot-path cases (run on the GPU box).
# usage: bash tools/sanitize_all.sh OUTDIR
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # tool case timeout
  local tool=$1 case=$2 to=$3
  echo "== $tool $case" | tee -a "$out/summary.txt"
  timeout "$to" $CS --tool "$tool" --error-exitcode 9 --print-limit 50 python tools/sanitize_case.py "$case" \
      > "$out/${tool}_${case}.log" 2>&1
  local rc=$?
  tail -n 3 "$out/${tool}_${case}.log" | tee -a "$out/summary.txt"
  echo "rc=$rc" | tee -a "$out/summary.txt"
}
python tools/sanitize_case.py c1 > /dev/null 2>&1   # warm (page in torch)
for c in c1 c2 g3_700 g4_300 batched ipm pipeline; do run memcheck $c 900; done
for c in c1 g3_700 batched ipm; do run racecheck $c 1200; done
for c in c1 g3_700 batched ipm; do run synccheck $c 900; done
run initcheck c1 600
