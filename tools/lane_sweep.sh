#!/bin/bash
# Concurrency sweep of the K-column THROUGHPUT block solve on config 2:
# lanes x block width x tail variant (tools/batch_timing.py, bounded cycles).
#   bash tools/lane_sweep.sh [max_cycles]
MC=${1:-12}
run() {  # lanes block env...
  local lanes=$1 block=$2; shift 2
  echo "== lanes $lanes block $block $*"
  env LANES=$lanes "$@" python tools/batch_timing.py 2 $block 2 $MC 2>&1 | grep -E "rep 1|rror"
}
for spec in "8 32 16" "8 32 8" "8 32 4" "16 32 8" "16 32 4" "4 64 16" "4 64 8" "8 64 4" "2 128 16" "4 128 8"; do
  set -- $spec
  run $1 $2 LAMG_BATCH_CTAS=$3
done
for small in 4096 8192 16384; do
  for kc in 1 2 4; do
    run 8 32 LAMG_BATCH_TAIL=subtree LAMG_BATCH_SMALL=$small LAMG_BATCH_KC=$kc
  done
done
run 16 32 LAMG_BATCH_TAIL=subtree LAMG_BATCH_SMALL=8192 LAMG_BATCH_KC=4
run 16 32 LAMG_BATCH_TAIL=subtree LAMG_BATCH_SMALL=16384 LAMG_BATCH_KC=4
run 1 32 LAMG_BATCH_CTAS=16
run 1 32 LAMG_BATCH_TAIL=subtree LAMG_BATCH_SMALL=4096 LAMG_BATCH_KC=1
run 1 32 LAMG_BATCH_TAIL=subtree LAMG_BATCH_SMALL=16384 LAMG_BATCH_KC=1
run 1 32 LAMG_BATCH_TAIL=subtree LAMG_BATCH_SMALL=16384 LAMG_BATCH_KC=4
