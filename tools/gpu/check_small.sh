cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_slot_gpu.py tests/test_pack_gpu.py -m gpu -q --tb=short -p no:cacheprovider 2>&1 | tail -2
for P in 45864 22932 11466 5733; do python tools/quick_bench.py 16 16 $P fp32 20 2>&1 | grep -v Warn | tail -1; done
