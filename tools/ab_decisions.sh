# A/B for numerics-changing variants (dev tool, under gpurun): decision agreement
# with build/var/old, timings, and parity at scale against the FP64-exact kernel
set -u
python tools/dump_outputs.py gpurun_out/ab_new.npz 2>&1 | grep -v Warn
ISINGLINK_B200_LIB=build/var/old/libisinglink_b200.so python tools/dump_outputs.py gpurun_out/ab_old.npz 2>&1 | grep -v Warn
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/ab_new.npz'); b=np.load('gpurun_out/ab_old.npz')
for k in a:
    if k.endswith('x_idx'):
        print(k, 'RE decisions identical: %.5f' % (a[k]==b[k]).reshape(a[k].shape[0],-1).all(1).mean())
    if k.endswith('energy'):
        print(k, 'mean energy new %.6f old %.6f' % (a[k].mean(), b[k].mean()))
    if k.endswith('diverged'):
        print(k, 'mean diverged new %.4f old %.4f' % (a[k].mean(), b[k].mean()))
PY
for v in old default old default; do if [ $v = default ]; then L=paper_2510_01579_b200/_lib/libisinglink_b200.so; else L=build/var/$v/libisinglink_b200.so; fi; ISINGLINK_B200_LIB=$L python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | sed "s/^/$v /"; done
python tools/quick_bench.py 8 16 45864 fp32 3 2>&1 | grep -v Warn
python tools/parity_scale.py 8192 2>&1 | grep -v Warn
