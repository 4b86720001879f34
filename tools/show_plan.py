"""Print the device program plan of a formula (needs a GPU).
  python tools/show_plan.py [chain|c3|c1]"""
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

from paper_2010_07284_b200 import PixelKind  # noqa: E402
from paper_2010_07284_b200 import synth as S  # noqa: E402
from paper_2010_07284_b200.executor import Program  # noqa: E402
from paper_2010_07284_b200.imgql import compile_text  # noqa: E402

C1 = ('load img = "img.png"\nlet a = img >. 62258\nlet b = img >. 56360\n'
      'save "out.png" reach(near(near(near(near(a & !b)))), b)\n')  # bench.py C1_SPEC
which = sys.argv[1] if len(sys.argv) > 1 else "chain"
if which == "chain":
    g, name, img = compile_text(S.near_reach_chain(6)), "img.png", S.blob_noise(1024, 1024, 1)
elif which == "c3":
    g, name = compile_text(S.SEGMENTATION_SPEC), "slices.png"
    img = np.stack([S.blob_noise(240, 240, 100 + i) for i in range(155)])
else:
    g, name, img = compile_text(C1), "img.png", S.blob_noise(256, 256, 1)
p = Program(g)
p.set_input_host(name, img, PixelKind.U16)
p.run(label_cse=False)
print(p.plan)
