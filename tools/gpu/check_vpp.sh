cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_slot_gpu.py tests/test_multi_gpu.py tests/test_baseline_curves.py tests/test_helpers_gpu.py tests/test_pack_gpu.py tests/test_philox_gpu.py -m gpu -q --tb=short -p no:cacheprovider 2>&1 | tail -4
python tools/vpp_prof.py 2>&1 | tail -1
python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn | tail -1
