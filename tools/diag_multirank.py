import sys
import numpy as np
sys.path.insert(0, '.')
from oracle import oracle as O
from tests.test_gpu_multirank import make
g = (16, 12, 8, 2e-9, 2e-9, 2e-9)
m = O.random_unit_field(16 * 12 * 8, 8e5, 23)
for trial in range(3):
    for mode in ['6', '1x6']:
        one, many = make(g, 64, 1), make(g, 64, 2)
        one.set_m(m); many.set_m(m)
        if mode == '6':
            a = many.step(6, return_all=True); b = one.step(6, return_all=True)
        else:
            a = np.array([many.step(1) for _ in range(6)]); b = np.array([one.step(1) for _ in range(6)])
        print(trial, mode, 'max torque diff', np.abs(a - b).max(), 'M diff', np.abs(many.get_m() - one.get_m()).max())
