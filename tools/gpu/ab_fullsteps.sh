# A/B of the refresh precision switch (ISINGLINK_FULL_STEPS): slot time + parity against fp64_exact
cd $GRAFT_REPO_ROOT
for k in "$@"; do
  echo "== full_steps=$k"
  ISINGLINK_FULL_STEPS=$k python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | tail -1
  ISINGLINK_FULL_STEPS=$k python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn | tail -1
  ISINGLINK_FULL_STEPS=$k timeout 600 python tools/parity_scale.py ${PAR_P:-16384} 2>&1 | grep -v Warn
done
