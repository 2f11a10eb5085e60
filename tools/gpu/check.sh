# parity subset touching the front end and the anneal + quick slot timings
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_slot_gpu.py tests/test_api_gpu.py tests/test_baseline_curves.py tests/test_multi_gpu.py -m gpu -q -s --tb=short -p no:cacheprovider > gpurun_out/check_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check_tests.log
grep -E "energy<=|passed|failed|Error" gpurun_out/check_tests.log | tail -12
for p in fp32 mixed; do python tools/quick_bench.py 16 16 45864 $p 5 2>&1 | grep -v Warn | tail -1; done
python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn | tail -1
