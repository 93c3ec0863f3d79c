for r in 1 2; do for o in 5 4; do
PDILQR_OCC_LS=$o SWEEP_CONFIGS="[{\"fold\":4,\"ls\":$o}]" timeout 200 python scripts/sweep_step.py
done; done
timeout 600 python -m pytest tests/test_gpu_srbd.py tests/test_gpu_solve.py tests/test_gpu_closed_loop.py -q -x 2>&1 | tail -2
