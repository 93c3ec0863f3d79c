for env in "PDILQR_SCAN_KS=1" "PDILQR_SCAN_KS=0" "PDILQR_KS_SPLIT=0"; do
  echo "== $env"; env $env timeout 300 python -m pytest tests/test_gpu_solve.py -q -x 2>&1 | tail -2
done
