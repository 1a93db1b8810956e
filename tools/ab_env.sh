#!/bin/bash
# A/B timing of the candidate kernel under environment overrides (same box, alternating).
#   tools/ab_env.sh "<config> <K>" "ENV1=a ENV2=b" "ENV1=c" ...
# Each variant runs prof_balance.py (3 reps) twice, interleaved; prints the last rep's ms.
set -u
read -r CFG K <<< "$1"
shift
for round in 1 2; do
  for v in "$@"; do
    ms=$(env $v DFLOP_DEBUG=1 python tools/prof_balance.py --config "$CFG" --K "$K" --reps 3 2>&1 \
         | tee -a gpurun_out/ab_raw.log | grep '^rep 2' | awk '{print $5}')
    echo "cfg$CFG K=$K [$v] round $round: $ms ms"
  done
done
