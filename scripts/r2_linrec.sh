#!/bin/bash
# A/B of the record-fed fold (PDILQR_LINREC) and its occupancy, then the SRBD step parity tests.
mkdir -p gpurun_out
for lr in 0 1; do for o in 4 5 6; do
  [ $lr = 0 ] && [ $o != 4 ] && continue
  PDILQR_LINREC=$lr SWEEP_CONFIGS="[{\"fold\":$o,\"ls\":4}]" timeout 200 python scripts/sweep_step.py 2>&1 | sed "s/^/linrec=$lr /"
done; done | tee gpurun_out/linrec_sweep.txt
timeout 900 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_solve.py tests/test_gpu_closed_loop.py -q -x 2>&1 | tail -5
