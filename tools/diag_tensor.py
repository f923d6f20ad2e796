import sys, numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from tests.helpers import engine_sim
from tests.test_gpu_parity import spec_of
for g in [(8, 8, 8, 2e-9, 2e-9, 2e-9), (128, 32, 1, 3.90625e-9, 3.90625e-9, 3e-9),
          (40, 20, 8, 0.9765625e-9, 0.9765625e-9, 0.75e-9), (24, 24, 24, 3.90625e-9, 3.90625e-9, 3.90625e-9),
          (5, 3, 2, 1e-9, 2e-9, 3e-9), (300, 2, 2, 1e-9, 1e-9, 1e-9)]:
    dev = engine_sim(spec_of(g), 64).demag_octant()
    tr = O.tensor_octant(*g, which="quad")
    ref = O.tensor_octant(*g, which="ref")
    for c in range(6):
        sc = np.max(np.abs(tr[c]))
        big = np.abs(tr[c]) > 1e-9 * sc
        e = np.abs(dev[c] - tr[c]); er = np.abs(ref[c] - tr[c])
        rel = np.where(big, e / np.maximum(np.abs(tr[c]), 1e-300), 0)
        relr = np.where(big, er / np.maximum(np.abs(tr[c]), 1e-300), 0)
        i = np.unravel_index(np.argmax(rel), rel.shape)
        print(g[:3], c, f"dev maxrel {rel.max():.2e} at kji={i} | maxabs/scale {e.max()/sc:.2e} | ref maxrel {relr.max():.2e} abs/scale {er.max()/sc:.2e}")
