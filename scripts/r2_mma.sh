#!/bin/bash
# mma.sync 3xTF32 products of the large-n fold: timing of configs 4/5 (SIMT vs MMA) and large-path parity
mkdir -p gpurun_out
for mm in 0 1; do PDILQR_BIG_MMA=$mm timeout 300 python scripts/bench_big.py 2>&1 | sed "s/^/mma=$mm /"; done | tee gpurun_out/mma_big.txt
timeout 900 python -m pytest tests/test_gpu_big.py tests/test_gpu_multi.py -q -x -k "mma or not simt and not tc" 2>&1 | tail -4
