timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
SWEEP_CONFIGS='[{"fold":4,"ls":4}]' python scripts/sweep_step.py
PDILQR_FUSED=1 SWEEP_CONFIGS='[{"fold":4,"ls":4}]' python scripts/sweep_step.py
LAT_N=50,1000 LAT_CHUNK=0 python scripts/lat_breakdown.py
