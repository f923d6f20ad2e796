"""Per-pass device times at C4 with the local terms switched off one by one
(how much of K5 is the H_eff/LLG epilogue): python tools/k5_probe.py"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1406_7459_b200 as E

g = E.Grid(512, 512, 64, 2.5e-9, 2.5e-9, 2.5e-9)
for name, mat, f in [
    ("all terms", E.Material(A=1.3e-11, Ku=4e4, Ms=8e5, alpha=0.02), E.FieldConfig(True, True, True, True, (1e4, 0, 0))),
    ("no exchange", E.Material(A=0.0, Ku=4e4, Ms=8e5, alpha=0.02), E.FieldConfig(True, True, True, True, (1e4, 0, 0))),
    ("demag only", E.Material(A=0.0, Ku=0.0, Ms=8e5, alpha=0.02), E.FieldConfig(True, True, True, True, (0, 0, 0))),
]:
    sim = E.Simulation(g, mat, f, E.StepperConfig(dt=1e-14), precision=32, init_direction=(3 ** -0.5,) * 3)
    sim.step_async(20); sim.sync()
    acc = np.zeros(7)
    for _ in range(20):
        acc += sim.step_timing()
    print(f"{name:12s}", " ".join(f"{v:.4f}" for v in acc[:6] / 20))
    sim.close()
