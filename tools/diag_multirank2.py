import numpy as np, sys
sys.path.insert(0, '.')
from tests.test_gpu_multirank import make, GRIDS, MS
from oracle import oracle as O
for g in GRIDS:
  for prec in (32, 64):
    for world in (2, 4):
        if g[2] % world: continue
        m = O.random_unit_field(g[0] * g[1] * g[2], MS, 23)
        one, many = make(g, prec, 1), make(g, prec, world)
        one.set_m(m); many.set_m(m)
        d1 = np.abs(many.demag_field() - one.demag_field()).max()
        e1 = np.abs(many.effective_field() - one.effective_field()).max()
        t = np.abs(many.step(6, return_all=True) - one.step(6, return_all=True)).max()
        mm = np.abs(many.get_m() - one.get_m()).max()
        print(g[:3], prec, world, 'demag', d1, 'heff', e1, 'torque', t, 'm', mm, flush=True)
