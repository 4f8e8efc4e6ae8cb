#!/bin/bash
# wave-round parameter sweep (rollout 16K / 64K): ring depth K (library builds) x switch threshold
for lib in build_ab/libK8.so build_ab/libK16.so; do
  for sw in 4096 8192 16384; do
    echo "lib=$lib switch=$sw $(PPG_LIB=$PWD/$lib PPG_WAVE_SWITCH=$sw python tools/wave_ab.py 2>&1 | tail -1)"
  done
done
echo "barrier: $(PPG_LIB=$PWD/build_ab/libK8.so PPG_WAVE=0 python tools/wave_ab.py 2>&1 | tail -1)"
