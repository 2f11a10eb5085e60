# tcgen05 vs mma.sync anneal (dev tool, run under gpurun)
set -u
timeout 300 env ISINGLINK_UMMA=1 python tools/dump_outputs.py gpurun_out/u_new.npz 2>&1 | grep -v Warn | tail -5
timeout 300 env ISINGLINK_UMMA=0 python tools/dump_outputs.py gpurun_out/u_old.npz 2>&1 | grep -v Warn | tail -5
python - <<'PY'
import numpy as np, os
if os.path.exists('gpurun_out/u_new.npz'):
    a=np.load('gpurun_out/u_new.npz'); b=np.load('gpurun_out/u_old.npz')
    for k in a:
        if k.endswith('x_idx'):
            same=(a[k]==b[k]).reshape(a[k].shape[0],-1).all(1).mean()
            print(k, 'RE decisions identical: %.4f' % same)
        elif k.endswith('energy'):
            print(k, 'mean energy new %.6f old %.6f  new<=old %.4f' % (a[k].mean(), b[k].mean(), (a[k]<=b[k]+1e-12).mean()))
PY
for u in 0 1; do timeout 300 env ISINGLINK_UMMA=$u python tools/quick_bench.py 16 16 45864 fp32 5 2>&1 | grep -v Warn | sed "s/^/umma=$u /"; done
for u in 0 1; do timeout 300 env ISINGLINK_UMMA=$u python tools/quick_bench.py 16 16 45864 tf32 3 2>&1 | grep -v Warn | sed "s/^/umma=$u /"; done
timeout 900 env ISINGLINK_UMMA=1 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
