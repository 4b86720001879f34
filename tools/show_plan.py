import sys; sys.path.insert(0,'.')
from paper_2010_07284_b200 import synth as S
from paper_2010_07284_b200.executor import Program
from paper_2010_07284_b200.imgql import compile_text
from paper_2010_07284_b200 import PixelKind
import numpy as np
g = compile_text(S.near_reach_chain(6))
p = Program(g)
p.set_input_host("img.png", S.blob_noise(1024, 1024, 1), PixelKind.U16)
p.run(label_cse=False)
print(p.plan)
