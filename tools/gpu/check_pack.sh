# packed (n_anneals <= 8) anneal: bit-identity tests + parity subset + replica-sweep timings
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_pack_gpu.py tests/test_gpu_parity.py tests/test_full_slot_gpu.py tests/test_api_gpu.py tests/test_baseline_curves.py tests/test_padding_counts_gpu.py -m gpu -q -s --tb=short -p no:cacheprovider > gpurun_out/check_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/check_tests.log
grep -E "packed ==|passed|failed|Error|assert" gpurun_out/check_tests.log | tail -20
for na in 8 16 32; do python tools/quick_bench.py 16 64 45864 fp32 3 $na 2>&1 | grep -v Warn | tail -1; done
ISINGLINK_PACK=0 python tools/quick_bench.py 16 64 45864 fp32 3 8 2>&1 | grep -v Warn | tail -1 | sed 's/^/[padded] /'
for na in 8 16; do python tools/quick_bench.py 8 16 45864 fp32 3 $na 2>&1 | grep -v Warn | tail -1; done
python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1
