cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
  ISINGLINK_B200_LIB=build/var/old/libisinglink_b200.so python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1 | sed 's/^/[old] /'
  python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1 | sed 's/^/[fused] /'
  ISINGLINK_FUSED_SELECT=0 python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1 | sed 's/^/[sep] /'
done
