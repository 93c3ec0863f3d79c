mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
TAG=${TAG:-r1_v8} bash scripts/profile_round.sh > gpurun_out/profile_round.log 2>&1
tail -c 300 gpurun_out/bench.log
