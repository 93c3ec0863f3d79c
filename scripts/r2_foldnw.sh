#!/bin/bash
# A/B of instances per warp (PDILQR_FOLD_NW) of the two-rows-per-lane fold, then the step parity tests.
mkdir -p gpurun_out
for nw in 4 5; do
  PDILQR_FOLD_NW=$nw SWEEP_CONFIGS='[{"fold":5,"ls":4}]' timeout 200 python scripts/sweep_step.py 2>&1 | sed "s/^/fold_nw=$nw /"
done | tee gpurun_out/foldnw_sweep.txt
PDILQR_FOLD_NW=${TEST_NW:-5} timeout 900 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_solve.py tests/test_gpu_closed_loop.py -q -x 2>&1 | tail -3
