#!/bin/bash
# A/B of the record-fed fold layouts (PDILQR_FOLD_MODE 0 / 1 / 2), then the step parity tests.
mkdir -p gpurun_out
for fm in 0 2; do
  PDILQR_FOLD_MODE=$fm SWEEP_CONFIGS='[{"fold":5,"ls":4}]' timeout 200 python scripts/sweep_step.py 2>&1 | sed "s/^/fold_mode=$fm /"
done | tee gpurun_out/foldmode_sweep.txt
timeout 900 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_solve.py tests/test_gpu_closed_loop.py -q -x 2>&1 | tail -5
