#!/bin/bash
# wave budget sweep (projection iterations per env per wave)
for b in 96 160 256 400 640; do
  echo "budget=$b $(PPG_WAVE_BUDGET=$b python tools/wave_ab.py 2>&1 | tail -1)"
done
