timeout 600 python bench.py --config c5 --steps 2 --warmup 1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 ms/step', d['ms_per_step'])"
python - <<'PY'
import sys, time, torch
sys.path.insert(0,'.')
from paper_2010_07284_b200 import Device, reach, ccl
from paper_2010_07284_b200.pixlog import random_mask_device
dev = Device(0)
for n in (32768, 65536):
    m = random_mask_device(n, n, 0.5, 1, 0, dev); t = random_mask_device(n, n, 0.05, 2, 0, dev)
    reach(t, m, dev); dev.synchronize()
    t0 = time.perf_counter(); r = reach(t, m, dev); dev.synchronize(); print(n, 'reach ms', (time.perf_counter()-t0)*1e3)
PY
