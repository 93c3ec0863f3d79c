#!/bin/bash
# linearisation-record kernel variants (PDILQR_LIN_STAGED 1 = one thread per stage, 2 = two warps per 32 stages), step parity
mkdir -p gpurun_out
for v in 1 2; do
  PDILQR_LIN_STAGED=$v SWEEP_CONFIGS='[{"fold":5,"ls":4}]' timeout 200 python scripts/sweep_step.py 2>&1 | sed "s/^/lin=$v /"
done | tee gpurun_out/lin_sweep.txt
timeout 900 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_solve.py tests/test_gpu_closed_loop.py -q -x 2>&1 | tail -3
