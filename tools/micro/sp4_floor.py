"""SP4 (128x32x1) per-step time of the graph-launched step under configurations
that bound it from below: the production two-kernel step, the unfused
three-kernel step, and demag off (one kernel per step: the launch floor of a
graph node chain).  python tools/micro/sp4_floor.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1406_7459_b200 as E  # noqa: E402

g = E.Grid(128, 32, 1, 500e-9 / 128, 125e-9 / 32, 3e-9)
mat = E.Material(A=1.3e-11, Ku=0.0, Ms=8e5, alpha=0.02, easy_axis=(0.0, 0.0, 1.0))


def run(demag, steps=6400):
    sim = E.Simulation(g, mat, E.FieldConfig(True, True, demag, True, (1e4, 0.0, 0.0)), E.StepperConfig(dt=1e-14),
                       precision=32, init_direction=(3 ** -0.5,) * 3)
    s = torch.cuda.ExternalStream(sim.stream_handle())
    sim.step_async(128)
    sim.sync()
    sim.prepare_async(steps)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    sim.step_async(steps)
    b.record(s)
    sim.sync()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps * 1e3


mode = os.environ.get("MFD_FUSE_K1", "default")
print(f"fuse={mode} demag on : {run(True):.2f} us/step")
print(f"fuse={mode} demag off: {run(False):.2f} us/step")
