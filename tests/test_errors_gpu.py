"""Failure paths of the C ABI (SURVEY §5 "failure detection", §8(b) "Errors").

A kernel launch that fails must surface as a non-zero status with a CUDA
message -- never SLCS_OK with an unwritten output.  The library's fault
injection (SLCS_FAULT_LAUNCH=n: the n-th launch of the process requests an
impossible amount of shared memory) makes a real launch fail; the test runs in
a subprocess so the injected failure cannot leak into other tests.
"""
import os
import subprocess
import sys
import textwrap

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = textwrap.dedent("""
    import ctypes as C, json, sys
    import numpy as np
    sys.path.insert(0, {root!r})
    from paper_2010_07284_b200 import _lib
    L = _lib.load()
    ctx = C.c_void_p()
    assert L.slcs_ctx_create(0, None, C.byref(ctx)) == 0
    a = (np.arange(64 * 48) % 3 == 0).astype(np.uint8)
    out = {{}}
    img = C.c_void_p()
    # launch 1: the upload's pack kernel
    out["upload"] = L.slcs_image_upload(ctx, 0, 64, 48, 1, a.ctypes.data, C.byref(img))
    out["upload_msg"] = L.slcs_last_error().decode()
    if out["upload"] == 0:
        r = C.c_void_p()
        out["near"] = L.slcs_near(ctx, img, C.byref(r))   # launch 2
        out["near_msg"] = L.slcs_last_error().decode()
        r2 = C.c_void_p()
        out["after"] = L.slcs_near(ctx, img, C.byref(r2))  # launch 3: healthy again
        host = np.zeros(64 * 48, np.uint8)
        out["download"] = L.slcs_image_download(ctx, r2, host.ctypes.data, host.nbytes)
        out["after_ok"] = bool(host.sum() > 0)
    hb = np.zeros(64 * 48, np.uint8)
    out["h_dilate"] = L.slcs_h_dilate(ctx, a.ctypes.data, 64, 48, hb.ctypes.data)
    print(json.dumps(out))
""")


def _run(at):
    env = dict(os.environ, SLCS_FAULT_LAUNCH=str(at))
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    import json
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_failed_launch_returns_cuda_status():
    SLCS_ERR_CUDA = 5
    o = _run(2)  # the near kernel fails
    assert o["upload"] == 0
    assert o["near"] == SLCS_ERR_CUDA, o
    assert "kernel launch" in o["near_msg"] or "CUDA" in o["near_msg"], o
    # the failure is reported once; later calls on the same context work
    assert o["after"] == 0 and o["download"] == 0 and o["after_ok"], o
    assert o["h_dilate"] == 0, o


def test_failed_upload_pack_returns_cuda_status():
    o = _run(1)  # the upload's packing kernel fails
    assert o["upload"] == 5, o
    assert o["h_dilate"] == 0, o


def test_host_wrapper_failure_status():
    # launches: 1 upload pack, 2 near, 3 near, 4 download unpack, 5 the host
    # wrapper's upload pack
    o = _run(5)
    assert o["near"] == 0 and o["after"] == 0 and o["download"] == 0, o
    assert o["h_dilate"] == 5, o


BAND_SCRIPT = textwrap.dedent("""
    import ctypes as C, json, sys
    import numpy as np
    sys.path.insert(0, {root!r})
    from paper_2010_07284_b200 import _lib
    L = _lib.load()
    ctx = C.c_void_p()
    assert L.slcs_ctx_create(0, None, C.byref(ctx)) == 0
    w, h = 700, 300
    rng = np.random.default_rng(3)
    u = (rng.random((h, w)) < 0.5).astype(np.uint8)
    t = (rng.random((h, w)) < 0.03).astype(np.uint8)

    def attempt():
        codes = []
        du, dt = C.c_void_p(), C.c_void_p()
        codes.append(L.slcs_image_upload(ctx, 0, w, h, 1, u.ctypes.data, C.byref(du)))
        codes.append(L.slcs_image_upload(ctx, 0, w, h, 1, t.ctypes.data, C.byref(dt)))
        if any(codes):
            return codes, None
        import torch
        recb = torch.zeros(L.slcs_band_record_bytes(1, w), dtype=torch.uint8, device="cuda")
        out = torch.zeros((h, w), dtype=torch.int64, device="cuda")
        st, job, sel = C.c_void_p(), C.c_void_p(), C.c_void_p()
        rc = L.slcs_reach_prepare_labels(ctx, dt, du, C.byref(st))
        codes.append(rc)
        if rc == 0:
            rc = L.slcs_ccl_band_begin_reach(st, C.c_void_p(recb.data_ptr()), C.byref(job))
            codes.append(rc)
            codes.append(L.slcs_reach_finish(st, 0, C.byref(sel)))
            if rc == 0:
                hs = (C.c_longlong * 1)(h)
                codes.append(L.slcs_ccl_band_finish(job, 1, 0, C.c_void_p(recb.data_ptr()), hs,
                                                    C.c_void_p(out.data_ptr())))
                codes.append(L.slcs_ccl_job_destroy(job))
            codes.append(L.slcs_reach_state_destroy(st))
        torch.cuda.synchronize()
        return codes, out.cpu().numpy()

    first, _ = attempt()
    again, lab = attempt()
    print(json.dumps({{"first": first, "again": again, "labels": int(lab.max()) if lab is not None else -1}}))
""")


@pytest.mark.parametrize("at", [1, 3, 4, 5, 6, 7, 8, 9])
def test_band_reach_labels_launch_failures(at):
    """A failed launch anywhere in the shared reach + labels band sequence is a
    status code from the call that issued it; the objects still destroy cleanly
    and the next sequence on the same context succeeds."""
    env = dict(os.environ, SLCS_FAULT_LAUNCH=str(at))
    r = subprocess.run([sys.executable, "-c", BAND_SCRIPT.format(root=ROOT)], env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    import json
    o = json.loads(r.stdout.strip().splitlines()[-1])
    assert any(c != 0 for c in o["first"]), o          # the injected failure surfaced
    assert all(c == 0 for c in o["again"]), o          # and left the context usable
    assert o["labels"] > 0, o
