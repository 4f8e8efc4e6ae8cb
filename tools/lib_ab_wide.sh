#!/bin/bash
# wide-batch decision timings (tools/async_wide.py) for library variants
for r in 1 2; do for lib in "$@"; do
  echo "$lib $(PPG_LIB=$PWD/$lib python tools/async_wide.py 2>&1 | tail -1 | cut -c1-400)"
done; done
