"""Diagnostics: phase timeline of the fused reach kernels of a short config-2 chain
(run with SLCS_PHASE_TIMING=1; CUDA graph off so the per-launch timing works)."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2010_07284_b200 import PixelKind  # noqa: E402
from paper_2010_07284_b200 import synth as S  # noqa: E402
from paper_2010_07284_b200.executor import Program  # noqa: E402
from paper_2010_07284_b200.imgql import compile_text  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
p = Program(compile_text(S.near_reach_chain(8)))
p.set_input_host("img.png", S.blob_noise(n, n, 1), PixelKind.U16)
p.run(label_cse=False, cuda_graph=False)
p.run(label_cse=False, cuda_graph=False)
print(p.plan)
