# parity subset + quick slot timings for the default build and each named variant (build/var/<v>)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_slot_gpu.py tests/test_api_gpu.py tests/test_baseline_curves.py tests/test_multi_gpu.py -m gpu -q -s --tb=short -p no:cacheprovider > gpurun_out/check_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check_tests.log
grep -E "passed|failed|Error" gpurun_out/check_tests.log | tail -5
for rep in 1 2; do
for v in default "$@"; do
  if [ "$v" = default ]; then L=paper_2510_01579_b200/_lib/libisinglink_b200.so; else L=build/var/$v/libisinglink_b200.so; fi
  ISINGLINK_B200_LIB=$L python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"
  ISINGLINK_B200_LIB=$L python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"
done
done
