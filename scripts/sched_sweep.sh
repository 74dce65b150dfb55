#!/bin/bash
# K1 schedules side by side: default rule vs stream-K at k = 1..4 waves of CTA slots,
# on whole configs and the largest block of each partition (scripts/sched_compare.py).
# CFGS / SPLITS / SKS override the sets; output JSON lines on stdout.
CFGS=${CFGS:-"c2 c3 c4 c5"}
SPLITS=${SPLITS:-"1x1,2x1,1x2,4x1,2x2,1x4,8x1,4x2,2x4,1x8"}
SKS=${SKS:-default 1 2 3 4}
for sk in $SKS; do
  if [ "$sk" = default ]; then
    python scripts/sched_compare.py $CFGS --splits $SPLITS $EXTRA
  else
    SWDFT2D_K1_STREAMK=$sk python scripts/sched_compare.py $CFGS --splits $SPLITS $EXTRA
  fi
done
