import os, sys, subprocess
import numpy as np
sys.path.insert(0, ".")
from tests import inputs as gen
name, n = sys.argv[1], int(sys.argv[2])
scalars, grids, adjs = gen.family_inputs(name, n, seed=n, accumulate=True)
g = {k: v.astype(np.float32).astype(np.float64) for k, v in grids.items()}
a = {k: v.astype(np.float32).astype(np.float64) for k, v in adjs.items()}
outs = {}
np.savez('/tmp/in.npz', g=g, a=a, sc=scalars)
for v in ("5", "7"):
    code = f"""
import sys, numpy as np; sys.path.insert(0,'.')
from paper_1907_02818_b200 import api
d=np.load('/tmp/in.npz', allow_pickle=True)
g=d['g'].item(); a=d['a'].item(); sc=d['sc'].item()
r=api.run_program('{name}', {n}, sc, g, a, dtype='f32')
np.save('/tmp/out{v}.npy', r['c_b'])
"""
    subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SGB_STAR_KERNEL=v), check=True)
    outs[v] = np.load(f"/tmp/out{v}.npy")
d = np.abs(outs["5"] - outs["7"])
bad = np.argwhere(d > 1e-4)
print(name, n, "bad points", len(bad), "of", d.size)
if len(bad):
    print("planes", np.unique(bad[:, 0])[:40])
    print("rows", np.unique(bad[:, 1])[:40])
    print("cols", np.unique(bad[:, 2])[:40])
    for p in bad[:6]:
        print(p, outs["5"][tuple(p)], outs["7"][tuple(p)])
