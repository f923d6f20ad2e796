import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from tests.helpers import engine_sim
from tests.test_gpu_parity import spec_of

g = (8, 8, 1, 2e-9, 2e-9, 2e-9)
s = spec_of(g)
sim = engine_sim(s, 64)
m = O.random_unit_field(s.n, s.Ms, 3)
sim.set_m(m)
B2 = sim.debug_stage(2)
hx = 9
for c in range(6):
    oct6 = np.zeros((6, 1, 8, 8))
    oct6[c, 0, 0, 0] = 1.0
    sim.set_demag_octant(oct6)
    spec = sim.spectrum_octant()
    B3 = sim.debug_stage(3)
    print('comp', c, 'spectrum min/max per comp', [(round(spec[q].min(), 3), round(spec[q].max(), 3)) for q in range(6)])
    for q in range(3):
        r = B3[q, :, :, :hx] / np.where(np.abs(B2[q, :, :, :hx]) > 0, B2[q, :, :, :hx], 1)
        print('   out comp', q, 'ratio B3/B2 stats', np.round(np.abs(r).min(), 4), np.round(np.abs(r).max(), 4),
              'B3 max', np.abs(B3[q, :, :, :hx]).max(), 'B2 max', np.abs(B2[q, :, :, :hx]).max())
