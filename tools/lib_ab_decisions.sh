#!/bin/bash
# decision / rollout timings (tools/async_ab.py) for library variants: bash tools/lib_ab_decisions.sh a.so b.so ...
for r in 1 2; do for lib in "$@"; do
  echo "$lib $(PPG_LIB=$PWD/$lib PLANNER=device python tools/async_ab.py 2>&1 | tail -1 | cut -c1-330)"
done; done
