# A/B of build/var/old vs the default build on the non-headline modes (dev
# tool, run under gpurun): tf32, philox, VPP, 8x8 PACK, padded shapes
cd $GRAFT_REPO_ROOT
for v in old new; do
  L=build/var/$v/libisinglink_b200.so
  for shape in "16 16 45864 tf32 5" "16 16 45864 fp32 5 32 philox" "8 16 45864 fp32 5 8" "20 16 45864 fp32 3" "6 16 45864 fp32 3" "32 16 45864 fp32 2"; do
    ISINGLINK_B200_LIB=$L python tools/quick_bench.py $shape 2>&1 | grep -v Warn | tail -1 | sed "s/^/[$v] /"
  done
  ISINGLINK_B200_LIB=$L python tools/vpp_time.py 2>&1 | grep -v Warn | head -1 | sed "s/^/[$v] vpp /"
done
