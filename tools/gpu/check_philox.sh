cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_philox_gpu.py tests/test_pack_gpu.py tests/test_gpu_parity.py tests/test_full_slot_gpu.py tests/test_reference_suite_gpu.py tests/test_abi.py -m gpu -q -s --tb=short -p no:cacheprovider > gpurun_out/check_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check_tests.log
grep -E "philox|passed|failed|Error|assert" gpurun_out/check_tests.log | tail -20
for r in numpy philox; do python tools/quick_bench.py 16 16 45864 fp32 5 32 $r 2>&1 | grep -v Warn | tail -1; done
python tools/quick_bench.py 16 16 45864 fp64_exact 1 32 philox 2>&1 | grep -v Warn | tail -1
