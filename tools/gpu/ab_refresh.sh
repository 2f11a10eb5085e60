# A/B of refresh-pass variants: slot time + parity against fp64_exact at scale
cd $GRAFT_REPO_ROOT
[ "$MB" = 1 ] && ./tools/microbench/mma_kinds
for v in ${VARIANTS:-default} "$@"; do
  echo "== $v"
  if [ "$v" = default ]; then L=paper_2510_01579_b200/_lib/libisinglink_b200.so; else L=build/var/$v/libisinglink_b200.so; fi
  ISINGLINK_B200_LIB=$L python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1
  ISINGLINK_B200_LIB=$L python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn | tail -1
  ISINGLINK_B200_LIB=$L timeout 600 python tools/parity_scale.py 16384 2>&1 | grep -v Warn
done
