for r in 1 2; do for s in 0 1; do for f in m c; do echo "sched=$s flags=$f $(PPG_SLICE_FLAGS=$f PPG_SLICE_SCHED=$s python tools/e2e_ab.py 65536 2>&1 | tail -1 | cut -c1-200)"; done; done; done > gpurun_out/r2e_slices2.log
PPG_SLICE_FLAGS=c python -m pytest tests -m gpu -q -x -k "stream or pipelined or host" -p no:cacheprovider > gpurun_out/r2e_slices_tests.log 2>&1
