#!/bin/bash
# step time / offer volume vs the number of NN-descent sub-rounds
for k in 1 2 4 8; do
  echo "== ANNK_SUBROUNDS=$k"
  ANNK_SUBROUNDS=$k timeout 300 python tools/step_overhead.py 2>&1 | grep -E "^plain|^it1|^it2" | tail -3 | cut -c1-400
done
