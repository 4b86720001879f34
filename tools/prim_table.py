"""Print bench.py's per-primitive table (config-4 size by default) as JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2010_07284_b200 import Device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
dev = Device(0, stream=stream.cuda_stream)
t = (bench.primitive_table(dev, stream, 0, n=n) if n <= 16384 else
     bench.primitive_table(dev, stream, 0, n=n, reps=5, copies=2, labels=False))
print("copy ceiling", t["copy_ceiling_gbs"], "GB/s")
for k, v in t["ops"].items():
    print(f"{k:10s} {v['ms']:9.4f} ms {v['gbs']:8.1f} GB/s frac={v['frac']:.3f} launches={v['launches']}")
print(json.dumps(t))
