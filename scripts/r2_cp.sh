#!/bin/bash
# stance-compacted policy solve in the fold (PDILQR_FOLD_CP), then the SRBD parity tests incl. the fused variants
mkdir -p gpurun_out
for cp in 0 1; do
  PDILQR_FOLD_CP=$cp SWEEP_CONFIGS='[{"fold":5,"ls":4}]' timeout 200 python scripts/sweep_step.py 2>&1 | sed "s/^/cp=$cp /"
done | tee gpurun_out/cp_sweep.txt
timeout 900 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_solve.py tests/test_gpu_closed_loop.py -q -x 2>&1 | tail -3
PDILQR_FOLD_CP=0 timeout 900 python -m pytest tests/test_gpu_srbd.py -q -x -k "fused or 4096" 2>&1 | tail -2
