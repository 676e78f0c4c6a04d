cd $GRAFT_REPO_ROOT
timeout 120 python scripts/tc_check.py > gpurun_out/tc_check.log 2>&1; echo "tc_check rc=$?" >> gpurun_out/tc_check.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -rf > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/tc_check.log
