# A/B of library variants on the NT >= 5 register layouts (dev tool, run
# under gpurun): n_t = 20 / 24 / 28 / 32 slot timings.  Variants: $@
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  L=build/var/$v/libisinglink_b200.so
  for shape in "16 16 45864 fp32 3" "20 16 45864 fp32 2" "24 16 45864 fp32 2" "28 16 45864 fp32 2" "32 16 45864 fp32 2"; do
    ISINGLINK_B200_LIB=$L python tools/quick_bench.py $shape 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"
  done
done
