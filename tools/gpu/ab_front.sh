# A/B of library variants: per-kind ms from tools/quick_bench.py (16x16 and 8x8 slots)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_full_slot_gpu.py tests/test_api_gpu.py -m gpu -q --tb=short -p no:cacheprovider 2>&1 | tail -3
for rep in 1 2; do
for v in default "$@"; do
  echo "== $v"
  if [ "$v" = default ]; then
    python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1
    python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn | tail -1
  else
    ISINGLINK_B200_LIB=build/var/$v/libisinglink_b200.so python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1
    ISINGLINK_B200_LIB=build/var/$v/libisinglink_b200.so python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn | tail -1
  fi
done
done
