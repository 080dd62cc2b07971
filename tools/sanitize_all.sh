#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the small hot-path runs of
# tools/sanitize.py (cfg1 fp64 at K = 1, 2; a 256^2 config-3 crop fp32 at K = 1, 2, 4; a CPML
# channel with ROMs at K = 4).  Logs: gpurun_out/sanitize/<tool>_<case>_k<K>.log
set -u
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for ck in "cfg1 1" "cfg1 2" "cfg3crop 1" "cfg3crop 2" "cfg3crop 4" "pml 4"; do
    set -- $ck
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra --error-exitcode 9 python tools/sanitize.py --case $1 --k $2 \
      > $OUT/${tool}_$1_k$2.log 2>&1
    echo "$tool $1 K=$2 rc=$?" | tee -a $OUT/summary.txt
  done
done
