cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in default "$@"; do
  if [ "$v" = default ]; then L=paper_2510_01579_b200/_lib/libisinglink_b200.so; else L=build/var/$v/libisinglink_b200.so; fi
  ISINGLINK_B200_LIB=$L python tools/quick_bench.py 8 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"
  ISINGLINK_B200_LIB=$L python tools/quick_bench.py 8 4 45864 fp32 5 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"
done
done
