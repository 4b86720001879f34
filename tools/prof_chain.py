"""One C2 formula evaluation (label CSE + k_reach_chain) for ncu / timing."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_07284_b200 import Device, PixelKind  # noqa: E402
from paper_2010_07284_b200 import synth as S  # noqa: E402
from paper_2010_07284_b200.executor import Program  # noqa: E402
from paper_2010_07284_b200.imgql import compile_text  # noqa: E402

depth = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = Device(0)
img = S.blob_noise(4096, 4096, 1)
prog = Program(compile_text(S.near_reach_chain(depth)), dev)
prog.set_input_host("img.png", img, PixelKind.U16)
for _ in range(runs):
    prog.run(cuda_graph=False)
dev.synchronize()
print(prog.plan.splitlines()[:6])

if "--time" in sys.argv:
    import time
    prog.run()  # graph capture
    dev.synchronize()
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        prog.run()
    dev.synchronize()
    print(f"formula: {(time.perf_counter() - t0) / reps * 1e3:.3f} ms (host-timed, back to back)")
    prog.run(timeline=True)
    out = [i for i, t in enumerate(prog.graph.nodes) if t.opcode == "save"][0]
    tt = prog.task_time(prog.graph.nodes[out].deps[0])
    print(f"chain kernel step: {tt[1] - tt[0]:.3f} ms")
