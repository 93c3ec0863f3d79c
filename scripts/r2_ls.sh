#!/bin/bash
# line-search rewrite: occupancy sweep of k_srbd_fwd_ls, then the SRBD step / solve / closed-loop / latency parity tests
mkdir -p gpurun_out
for o in 4; do
  PDILQR_OCC_LS=$o SWEEP_CONFIGS="[{\"fold\":5,\"ls\":$o}]" timeout 200 python scripts/sweep_step.py 2>&1 | sed "s/^/occ_ls=$o /"
done | tee gpurun_out/ls_sweep.txt
timeout 1200 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_solve.py tests/test_gpu_closed_loop.py -q -x 2>&1 | tail -3
