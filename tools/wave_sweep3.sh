#!/bin/bash
# wave-round switch threshold x budget re-sweep (rollout 16K / 64K) with the early-decision asynchronous tail
for sw in 8192 12288 16384 24576 40000; do
  for b in 192 256 384; do
    echo "switch=$sw budget=$b $(PPG_WAVE_SWITCH=$sw PPG_WAVE_BUDGET=$b python tools/wave_ab.py 2>&1 | tail -1)"
  done
done
