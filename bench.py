#!/usr/bin/env python3
"""Headline benchmark: BASELINE.json config 2 -- the 1000-deep near/reach
chain on a 4096x4096 synthetic blob-noise image, one
formula evaluation per step, on the device-resident program path.

metric  Gpixel-ops/s = (primitive nodes x pixels) / device time
        (load/save/const excluded); ms_per_step = ms per formula.
value   inputs resident in HBM; L2 flushed (512 MiB write) before every step,
        timed per step with CUDA events on the program's ordering stream.
e2e     the same metric through the public API with HOST buffers: per step the
        u16 image is copied H2D from pinned memory into the program's input
        slot and the Bool result (1 B/px, reference layout) is copied D2H.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
Under torchrun every rank evaluates its own replica (config 2 does not shard:
"replicas only"); value is the whole-job aggregate, timed as the max
over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_PX = {"reach": 8.375, "near": 0.25, "threshold": 2.125}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--size", type=int, default=4096)
    p.add_argument("--depth", type=int, default=1000)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--ref-depth", type=int, default=20,
                   help="chain depth of one bounded CPU-reference sample (~10 s on 16 "
                        "threads; its per-node rate is within 4%% of the full depth-1000 "
                        "run, profiles/r01f_cpu_reference.json)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-primitives", action="store_true",
                   help="skip the per-primitive table at 16384^2 (config 4 size)")
    p.add_argument("--no-label-cse", dest="label_cse", action="store_false",
                   help="headline with label CSE off: every reach node labels its own "
                        "`through` (the reference's per-node work, reach.cpp:21) in one fused "
                        "cooperative launch per reach.  Default on: the 500 reaches of the "
                        "chain share one labelling of `through` (computed inside every timed "
                        "step) and run as ONE persistent launch (k_reach_chain)")
    p.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"],
                   help="BASELINE.json config: c2 (default, the headline) or the parity/"
                        "secondary workloads c1, c3 (sharded by slice under torchrun), c4")
    p.add_argument("--density", type=float, default=0.5, help="c4 mask density (headline)")
    p.add_argument("--c5-size", type=int, default=65536,
                   help="image side of the C5 sub-result (BASELINE: 65536)")
    p.add_argument("--no-extra", action="store_true",
                   help="headline only: skip the C3 / C4 / C5 / Fig. 3 sub-results")
    p.add_argument("--alt-steps", type=int, default=3,
                   help="steps for the secondary measurement with label CSE toggled")
    return p.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# BENCH_DIST_BACKEND=gloo (test only): run the N>1 code path with several ranks on
# one GPU (ranks share devices round-robin); the driver's runs use NCCL, one GPU each
DIST_BACKEND = os.environ.get("BENCH_DIST_BACKEND", "nccl")


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if DIST_BACKEND != "nccl":
        import torch
        local %= max(1, torch.cuda.device_count())
    return ws, rank, local


def init_dist(local):
    import torch
    if DIST_BACKEND == "nccl":
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.distributed.init_process_group(DIST_BACKEND)


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def profiled_traffic(kernel_prefix, kind="traffic"):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of a
    kernel from the newest committed ncu summary profiles/r*_<kind>_*.json
    (serialised ncu replay), with the file it came from; (None, None) if absent."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_{kind}_*.json")),
                   key=lambda f: os.path.basename(f), reverse=True)
    for f in files:
        try:
            with open(f) as fh:
                d = json.load(fh)
        except (OSError, ValueError):
            continue
        for per_csv in d.values():
            for name, row in per_csv.items():
                if name.split("::")[-1].startswith(kernel_prefix) and row.get("dram_bytes_per_launch"):
                    return row["dram_bytes_per_launch"], os.path.relpath(f, ROOT) + " [" + name + "]"
    return None, None


def cpu_reference_sample(size, seed, ref_depth, steps=1):
    """The reference's own executor (oracle/_ref) on a bounded chain sample;
    falls back to the C restatement when oracle/_ref is absent."""
    import oracle as O
    from paper_2010_07284_b200 import synth as S
    from paper_2010_07284_b200.imgql import STDLIB
    img = S.blob_noise(size, size, seed)
    spec = S.near_reach_chain(ref_depth)
    cores = os.cpu_count() or 1
    px = size * size
    nodes = 2 + ref_depth
    times = []
    if os.path.exists(O._REF):
        R = O.Reference(workers=cores)
        kind = "reference"
        for _ in range(steps):
            res = R.run(spec, {"img.png": img}, STDLIB)
            times.append(res["computation_ms"] / 1e3)
    else:
        kind = "port"
        cores = 1
        for _ in range(steps):
            t0 = time.perf_counter()
            b = O.threshold(0, img, 56360)
            x = O.threshold(0, img, 62258)
            for k in range(ref_depth):
                x = O.dilate(x) if k % 2 == 0 else O.reach(x, b)
            times.append(time.perf_counter() - t0)
    return {"times": times, "nodes": nodes, "px": px, "kind": kind, "cores": cores,
            "sample": f"near/reach chain depth {ref_depth} (+2 thresholds) at "
                      f"{size}x{size}, blob-noise seed {seed}, executor::run with "
                      f"{cores} workers"}


def run_reference_arm(args, ws, rank):
    if rank != 0:
        return
    from paper_2010_07284_b200 import synth as S  # noqa: F401
    for _ in range(args.warmup if args.warmup < 2 else 1):
        cpu_reference_sample(args.size, args.seed, args.ref_depth, 1)
    r = cpu_reference_sample(args.size, args.seed, args.ref_depth, args.steps)
    t = sum(r["times"])
    gpo = r["nodes"] * r["px"] * args.steps / t / 1e9
    ms = t / args.steps * 1e3
    line = {
        "impl": "reference", "metric": "Gpixel-ops/s", "value": gpo, "unit": "Gpixel-ops/s",
        "n_gpus": 0 if ws == 1 else ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8/u16 (integer-exact)", "data": "synthetic",
        "ms_per_formula_extrapolated": ms / r["nodes"] * (args.depth + 2),
        "config": {"workload": f"near/reach chain (BASELINE config 2) at {args.size}x{args.size}"
                               f"; each step a bounded sample of depth {args.ref_depth}",
                   "image": f"{args.size}x{args.size}", "depth": args.depth,
                   "sample_depth": args.ref_depth},
        "cpu_baseline": {"value": gpo, "unit": "Gpixel-ops/s", "cores": r["cores"],
                         "kind": r["kind"], "sample": r["sample"]},
        "e2e": {"value": gpo, "unit": "Gpixel-ops/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


PRIM_BYTES = {"threshold": 2.125, "not": 0.25, "and": 0.375, "or": 0.375, "near": 0.25,
              "interior": 0.25, "near^4": 0.25, "volume": 0.125, "ccl": 4.125, "reach": 8.375,
              "maxvol": 8.25}  # SURVEY.md §8d algorithmic bytes per pixel


def primitive_table(dev, stream, local, n=16384, reps=10, copies=8, labels=True):
    """Every primitive at BASELINE config 4's size (n x n) through the device
    program path (C ABI, CUDA graph): one program applies the primitive to
    `copies` distinct inputs (copies x the image > L2, and L2 is flushed by a
    512 MiB write before every rep), timed with CUDA events on the stream the
    program is ordered on; per-launch time = rep time / copies.  ccl, reach and
    maxvol (ms-scale) are timed per direct C-ABI call.  GB/s = SURVEY §8d
    algorithmic bytes / time."""
    import torch

    from paper_2010_07284_b200 import DeviceImage, PixelKind, ccl, maxvol, reach
    from paper_2010_07284_b200.executor import Program
    from paper_2010_07284_b200.imgql import compile_text
    from paper_2010_07284_b200.pixlog import random_mask_device

    peak, _ = measured_peak_gbs()
    g = torch.Generator(device=f"cuda:{local}")
    g.manual_seed(1)
    R = copies
    raws = [torch.randint(-32768, 32767, (n, n), dtype=torch.int16, device=f"cuda:{local}",
                          generator=g) for _ in range(R)]
    torch.cuda.synchronize()
    u16 = [DeviceImage.from_device(r.data_ptr(), PixelKind.U16, n, n, 1, dev) for r in raws]
    del raws
    A = [random_mask_device(n, n, 0.5, 10 + i, 0, dev) for i in range(R)]
    B = [random_mask_device(n, n, 0.41, 30 + i, 0, dev) for i in range(R)]
    t = random_mask_device(n, n, 0.05, 2, 0, dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    forms = {"threshold": ("u{i} >. 30000", True), "not": ("!a{i}", False),
             "and": ("a{i} & b{i}", False), "or": ("a{i} | b{i}", False),
             "near": ("near(a{i})", False), "interior": ("interior(a{i})", False),
             "near^4": ("near(near(near(near(a{i}))))", False), "volume": ("volume(a{i})", False)}

    def time_fn(fn, k):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(reps)]
        l0 = dev.launches
        for e0, e1 in ev:
            flush.zero_()
            e0.record(stream)
            fn()
            e1.record(stream)
        torch.cuda.synchronize()
        ms = statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev) / k
        return ms, (dev.launches - l0) / reps / k

    out = {}
    for name, (expr, is_u16) in forms.items():
        lines = []
        for i in range(R):
            lines.append(f'load u{i} = "u{i}"' if is_u16 else f'load a{i} = "a{i}"')
            if "b{i}" in expr:
                lines.append(f'load b{i} = "b{i}"')
            e = expr.format(i=i)
            lines.append(f'print "v{i}" {e}' if name == "volume" else f'save "o{i}" {e}')
        prog = Program(compile_text("\n".join(lines) + "\n"), dev)
        for i in range(R):
            if is_u16:
                prog.bind(f"u{i}", u16[i])
            else:
                prog.bind(f"a{i}", A[i])
                if "b{i}" in expr:
                    prog.bind(f"b{i}", B[i])
        prog.run()
        ms, per = time_fn(prog.run, R)
        out[name] = {"ms": ms, "launches": per, "plan": prog.plan.strip().splitlines()[:2]}
        del prog
    if labels:  # u32 labels need W*H < 2^32 - 1 (image.cpp:26-28)
        for name, fn in {"ccl": lambda: ccl.label(A[0], dev),
                         "reach": lambda: reach(t, A[0], dev),
                         "maxvol": lambda: maxvol(A[0], dev)}.items():
            ms, per = time_fn(fn, 1)
            out[name] = {"ms": ms, "launches": per}
    # same-size ceiling: a device copy of one bool image (read + write), timed the same way
    src = [torch.empty(n * n // 8, dtype=torch.uint8, device=f"cuda:{local}") for _ in range(R)]
    dst = [torch.empty_like(x) for x in src]

    def copies_fn():
        for x, y in zip(src, dst):
            y.copy_(x)
    copy_ms, _ = time_fn(copies_fn, R)
    copy_gbs = 2 * (n * n // 8) / (copy_ms / 1e3) / 1e9
    del src, dst
    for name, d in out.items():
        gbs = PRIM_BYTES[name] * n * n / (d["ms"] / 1e3) / 1e9
        d.update({"ms": round(d["ms"], 4), "gbs": round(gbs, 1), "frac": round(gbs / peak, 3),
                  "bytes_per_px": PRIM_BYTES[name]})
    del flush
    return {"image": f"{n}x{n}", "copy_ceiling_gbs": round(copy_gbs, 1),
            "copy_ceiling_note": "torch copy_ of one bool image (same bytes as ! / near), "
                                 "timed the same way: the achievable HBM rate at this size",
            "inputs": f"{R} distinct inputs per primitive: u16 uniform "
                                           "random (torch); randomMask density 0.5 / 0.41; "
                                           "reach target density 0.05",
            "timing": "CUDA events on the program stream around one graph replay of "
                      f"{R} independent applications, L2 flushed before each; ms = per "
                      "application", "peak_gbs": peak, "ops": out}


C1_SPEC = ('load img = "img.png"\nlet a = img >. 62258\nlet b = img >. 56360\n'
           'save "out.png" reach(near(near(near(near(a & !b)))), b)\n')


def formula_result(args, ws, rank, local, dev, stream, config):
    """c1 (256^2) and c3 (155 x 240^2 slices, segmentation spec; the
    slices are sharded over the ranks, no data-path collective).  The batched
    output is checked against the reference-pinned sha256
    (tests/golden/large_checksums.json) at N=1."""
    import hashlib

    import numpy as np
    import torch

    from paper_2010_07284_b200 import PixelKind
    from paper_2010_07284_b200 import synth as S
    from paper_2010_07284_b200.executor import Program
    from paper_2010_07284_b200.imgql import STDLIB, compile_text

    if config == "c1":
        spec, name, seeds, n = C1_SPEC, "img.png", [args.seed], 256
        workload = "BASELINE config 1: reach(near^4(a & !b), b) on a 256x256 blob-noise image"
    else:
        spec, name, n = S.SEGMENTATION_SPEC, "slices.png", 240
        all_seeds = list(range(100, 255))  # 155 slices
        per = (len(all_seeds) + ws - 1) // ws
        seeds = all_seeds[rank * per:(rank + 1) * per] or [100]
        workload = ("BASELINE config 3: segmentation spec maxvol(grow(hI,vI)) | surrounded(hI,vI) "
                    "over 155 blob-noise 240x240 slices (seeds 100..254), one batched program")
    imgs = np.stack([S.blob_noise(n, n, sd) for sd in seeds])
    graph = compile_text(spec)
    prim = sum(1 for t in graph.nodes if t.opcode not in ("load", "save", "const"))
    out_task = [i for i, t in enumerate(graph.nodes) if t.opcode == "save"][0]
    prog = Program(graph, dev)
    pin_in = torch.from_numpy(imgs if len(seeds) > 1 else imgs[0]).pin_memory()
    pin_out = torch.empty(tuple(pin_in.shape), dtype=torch.uint8).pin_memory()
    prog.set_input_host(name, pin_in.numpy(), PixelKind.U16)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    for _ in range(max(3, args.warmup)):
        prog.run()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    l0 = dev.launches
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for a, b in ev:
            flush.zero_()
            a.record(stream)
            prog.run()
            b.record(stream)
        torch.cuda.synchronize()
    launches = dev.launches - l0
    t = sum(a.elapsed_time(b) for a, b in ev) / 1e3
    units_local = prim * n * n * len(seeds)
    if ws > 1:
        tt = torch.tensor([t], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
        uu = torch.tensor([units_local], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(uu)
        units = float(uu.item())
    else:
        units = units_local
    value = units * args.steps / t / 1e9
    # e2e through the public API with host buffers
    t0 = time.perf_counter()
    for _ in range(args.steps):
        prog.set_input_host(name, pin_in.numpy(), PixelKind.U16)
        prog.run()
        prog.download(out_task, pin_out.numpy())
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if ws > 1:
        tt = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(tt.item())
    checksum_ok = None
    if config == "c3" and ws == 1:
        want = golden("c3", "batch_sha256")
        if want:
            checksum_ok = hashlib.sha256(pin_out.numpy().tobytes()).hexdigest() == want
            assert checksum_ok, "C3 segmentation output differs from the reference-pinned sha256"
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle as O
        if os.path.exists(O._REF):
            R = O.Reference(workers=os.cpu_count() or 1)
            if config == "c1":
                tcpu = R.run(spec, {name: imgs[0]}, STDLIB)["computation_ms"] / 1e3
                cpu = {"value": prim * n * n / tcpu / 1e9, "unit": "Gpixel-ops/s",
                       "cores": os.cpu_count(), "kind": "reference",
                       "sample": "the whole formula through executor::run", "ms": tcpu * 1e3}
            else:
                # the reference's executor on all 155 slices in ONE task graph (independent
                # sub-DAGs run concurrently on its worker pool, executor.cpp:220,259); it
                # has no maxvol, so the CPU spec is grow | surrounded
                lines = []
                for q in range(len(seeds)):
                    lines += [f'load s{q} = "s{q}.png"', f"let h{q} = intensity(s{q}) >. 62258",
                              f"let v{q} = intensity(s{q}) >. 56360",
                              f'save "o{q}.png" grow(h{q}, v{q}) | surrounded(h{q}, v{q})']
                cpu_spec = "\n".join(lines) + "\n"
                res = R.run(cpu_spec, {f"s{q}.png": imgs[q] for q in range(len(seeds))}, STDLIB)
                tcpu = res["computation_ms"] / 1e3
                cpu_prim = sum(1 for t in compile_text(cpu_spec).nodes
                               if t.opcode not in ("load", "save", "const"))
                cpu = {"value": cpu_prim * n * n / tcpu / 1e9, "unit": "Gpixel-ops/s",
                       "cores": os.cpu_count(), "kind": "reference",
                       "sample": f"grow | surrounded on all {len(seeds)} slices as one task "
                                 f"graph through executor::run ({cpu_prim} primitive nodes; "
                                 "maxvol has no reference)", "ms": tcpu * 1e3}
    return {
        "metric": "Gpixel-ops/s", "value": value, "unit": "Gpixel-ops/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong" if config == "c3" else "weak",
        "vs_baseline": None, "dtype": "u1/u16 (bit-packed integer)", "data": "synthetic",
        "config": {"workload": workload, "slices_per_rank": len(seeds), "image": f"{n}x{n}",
                   "primitive_nodes": prim, "l2": "flushed before every timed step",
                   "parallelism": f"slices sharded over {ws} rank(s)" if ws > 1 else "single"},
        "ms_per_formula": t / args.steps * 1e3,
        "gpu_launches": launches, "kernels_per_formula": prog.launches,
        "checksum_ok": checksum_ok, "clocks": clocks.summary(),
        "e2e": {"value": units * args.steps / e2e_s / 1e9, "unit": "Gpixel-ops/s",
                "h2d_bytes_per_step": int(pin_in.numel()) * 2,
                "d2h_bytes_per_step": int(pin_out.numel()),
                "ms_per_step": e2e_s / args.steps * 1e3},
        "cpu_baseline": cpu}


def c4_result(args, ws, rank, local, dev, stream, n=16384):
    """c4: CCL + reach on a 16384^2 random mask (device-generated randomMask stream),
    densities 0.41 / 0.5 / 0.7; labels and reach results checked
    against the reference-pinned sha256 at N=1."""
    import hashlib

    import torch

    from paper_2010_07284_b200 import ccl, reach
    from paper_2010_07284_b200.pixlog import random_mask_device

    mask = random_mask_device(n, n, args.density, 1, 0, dev)
    target = random_mask_device(n, n, 0.05, 2, 0, dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    for _ in range(max(2, args.warmup)):
        ccl.label(mask, dev)
        reach(target, mask, dev)
    torch.cuda.synchronize()
    ec = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    er = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    l0 = dev.launches
    with ClockSampler(local) as clocks:
        for (a, b), (c, d) in zip(ec, er):
            flush.zero_()
            a.record(stream)
            lab = ccl.label(mask, dev)
            b.record(stream)
            del lab
            flush.zero_()
            c.record(stream)
            r = reach(target, mask, dev)
            d.record(stream)
            del r
        torch.cuda.synchronize()
    tc = sum(a.elapsed_time(b) for a, b in ec) / 1e3 / args.steps
    tr = sum(a.elapsed_time(b) for a, b in er) / 1e3 / args.steps
    px = n * n
    # reference-pinned outputs of the timed kernels (the same inputs)
    checks = {}
    if n == 16384:
        for dens in (0.41, 0.5, 0.7):
            want = golden("c4", f"d{dens}")
            if not want:
                continue
            m2 = random_mask_device(n, n, dens, 1, 0, dev)
            lab = ccl.label(m2, dev).numpy()
            rr = reach(target, m2, dev).numpy()
            checks[str(dens)] = (hashlib.sha256(lab.tobytes()).hexdigest() == want["ccl_sha256"]
                                 and hashlib.sha256(rr.tobytes()).hexdigest() ==
                                 want["reach_sha256"])
            del lab, rr, m2
        assert all(checks.values()), f"C4 outputs differ from the reference: {checks}"
    # SURVEY §8(d) C4 densities: the other two masks, same timing (not in `value`)
    sweep = {}
    for dens in (0.41, 0.5, 0.7):
        if abs(dens - args.density) < 1e-9:
            sweep[str(dens)] = {"ccl_ms": tc * 1e3, "reach_ms": tr * 1e3}
            continue
        m2 = random_mask_device(n, n, dens, 1, 0, dev)
        for _ in range(2):
            ccl.label(m2, dev)
            reach(target, m2, dev)
        tcs, trs = [], []
        for _ in range(args.steps):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            flush.zero_()
            ev[0].record(stream)
            lab = ccl.label(m2, dev)
            ev[1].record(stream)
            del lab
            flush.zero_()
            ev[2].record(stream)
            r = reach(target, m2, dev)
            ev[3].record(stream)
            del r
            torch.cuda.synchronize()
            tcs.append(ev[0].elapsed_time(ev[1]))
            trs.append(ev[2].elapsed_time(ev[3]))
        sweep[str(dens)] = {"ccl_ms": sum(tcs) / len(tcs), "reach_ms": sum(trs) / len(trs)}
        del m2
    # e2e through the reference-facing host wrappers (kernels/ccl/reach signatures,
    # slcs_h_*): pinned 1 B/px masks in, u32 labels and 1 B/px reach result out
    e2e = None
    if not args.no_e2e:
        import ctypes as C

        from paper_2010_07284_b200 import _lib
        from paper_2010_07284_b200.pixlog import _check as _check_rc
        L = _lib.load()
        pin_m = torch.empty((n, n), dtype=torch.uint8).pin_memory()
        pin_t = torch.empty((n, n), dtype=torch.uint8).pin_memory()
        pin_lab = torch.empty((n, n), dtype=torch.int32).pin_memory()
        pin_r = torch.empty((n, n), dtype=torch.uint8).pin_memory()
        pin_m.copy_(torch.from_numpy(mask.numpy()))
        pin_t.copy_(torch.from_numpy(target.numpy()))

        def e2e_step():
            _check_rc(L.slcs_h_ccl_label(dev.handle, C.c_void_p(pin_m.data_ptr()), n, n,
                                         C.c_void_p(pin_lab.data_ptr())))
            _check_rc(L.slcs_h_reach(dev.handle, C.c_void_p(pin_t.data_ptr()),
                                     C.c_void_p(pin_m.data_ptr()), n, n,
                                     C.c_void_p(pin_r.data_ptr())))

        e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_s = (time.perf_counter() - t0) / args.steps
        e2e = {"value": 2 * px / e2e_s / 1e9, "unit": "Gpixel-ops/s",
               "h2d_bytes_per_step": 3 * px, "d2h_bytes_per_step": 5 * px,
               "ms_per_step": e2e_s * 1e3,
               "timing": "host wall clock, synced (slcs_h_ccl_label + slcs_h_reach)"}
        del pin_m, pin_t, pin_lab, pin_r
    peak, pk = measured_peak_gbs()
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        import oracle as O
        if os.path.exists(O._REF):
            # the full-size workload's ccl::label, once (~15 s on 16 threads,
            # profiles/r01f_cpu_reference.json); reach is the same labelling + 4 passes
            R = O.Reference(workers=os.cpu_count() or 1)
            a = O.random_mask(n, n, args.density, O.Rng(1))
            t0 = time.perf_counter()
            R.ccl_label(a)
            t_cpu = time.perf_counter() - t0
            cpu = {"value": n * n / t_cpu / 1e9, "unit": "Gpixel-ops/s", "cores": os.cpu_count(),
                   "kind": "reference", "sample": f"ccl::label on the {n}x{n} random mask "
                                                  f"(density {args.density}), one call",
                   "ms": t_cpu * 1e3}
    # DRAM bytes of one ccl::label (its four kernels) from the newest committed
    # 16384^2 ncu breakdown (--cache-control none), or null
    ccl_traffic, ccl_src = None, None
    if n == 16384:
        parts = [profiled_traffic(k, "kernels_c4") for k in
                 ("k_tile_local<0", "k_tile_merge", "k_root_flatten", "k_tile_labels")]
        if all(t for t, _ in parts):
            ccl_traffic = sum(t for t, _ in parts)
            ccl_src = parts[0][1].split(" [")[0] + " (sum of the four ccl kernels)"
    if True:
        return ({
            "metric": "Gpixel-ops/s", "value": 2 * px / (tc + tr) / 1e9, "unit": "Gpixel-ops/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": (tc + tr) * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u1 -> u32 labels", "data": "synthetic",
            "config": {"workload": f"BASELINE config 4: ccl::label + reach on a {n}x{n} random "
                                   f"mask, density {args.density} (target density 0.05)",
                       "ccl_ms": tc * 1e3, "reach_ms": tr * 1e3, "densities": sweep},
            "gpu_launches": dev.launches - l0, "clocks": clocks.summary(),
            "roofline": {"bound": "hbm", "kernel": "ccl::label (tile-local UF, merge, flatten, "
                                                   "labels)",
                         "achieved": 4.125 * px / tc / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": 4.125 * px / tc / 1e9 / peak, "traffic": ccl_traffic,
                         "traffic_source": ccl_src, "peak_source": pk,
                         "note": "not HBM-bound: k_tile_local (~70 % of the ccl) is issue-bound "
                                 "(~84 % of issue slots busy at 13.8 active threads per warp "
                                 "instruction, 305 MB DRAM per launch; "
                                 "profiles/r02i_ncu_tile_local_full.txt); the union count per "
                                 "run is near its floor (DESIGN.md section 12)"},
            "checksum_ok": checks or None, "e2e": e2e, "cpu_baseline": cpu})


def c5_result(args, ws, rank, local, dev, stream, n=65536):
    """c5: a 65536^2 random mask in row bands, one per rank (the image is fixed ->
    strong scaling).  Per step: near^4 (k-row NCCL halo exchange read in place),
    volume (device all-reduce), reach (device cross-band merge of all-gathered
    border records) and ccl::label as global 64-bit labels (device merge +
    relabel).  At N=1, 65536^2 labels do not fit the reference's 32-bit packing
    (image.cpp:26-28): the labels run as two in-process bands."""
    import torch

    from paper_2010_07284_b200.bands import (LocalGroup, SoloComm, TorchComm, band_rows,
                                             near_banded, reach_ccl_banded, volume_banded)
    from paper_2010_07284_b200.pixlog import random_mask_device

    r0, r1 = band_rows(n, ws, rank)
    mask = random_mask_device(n, r1 - r0, 0.5, 1, r0, dev)
    target = random_mask_device(n, r1 - r0, 0.05, 2, r0, dev)
    comm = TorchComm() if ws > 1 else SoloComm()
    # reach(target, mask) and ccl::label(mask) share one labelling of the band
    # (reach_ccl_banded); at N=1, 65536^2 labels do not fit 32-bit keys, so both
    # run as two in-process bands
    if ws == 1 and n * n >= 0xFFFFFFFE:
        halves = [(random_mask_device(n, b - a, 0.05, 2, a, dev),
                   random_mask_device(n, b - a, 0.5, 1, a, dev))
                  for a, b in (band_rows(n, 2, 0), band_rows(n, 2, 1))]

        def reach_labels():
            return LocalGroup(2).run(lambda c, b: reach_ccl_banded(c, b[0], b[1]), halves)
    else:
        def reach_labels():
            return reach_ccl_banded(comm, target, mask)

    def step():
        x = near_banded(comm, mask, 4)
        v = volume_banded(comm, x)
        rl = reach_labels()
        return v, rl

    vol = None
    for _ in range(max(3, args.warmup)):
        vol = step()[0]
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = dev.launches
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    steps = max(1, min(args.steps, 5))
    with ClockSampler(local) as clocks:
        e0.record(stream)
        for _ in range(steps):
            step()
        e1.record(stream)
        dev.synchronize()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
    if ws > 1:
        tt = torch.tensor([t], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t = float(tt.item())
    ops = 4 + 1 + 1 + 1
    return {
        "metric": "Gpixel-ops/s", "value": ops * n * n * steps / t / 1e9,
        "unit": "Gpixel-ops/s", "n_gpus": ws, "steps": steps, "warmup": max(3, args.warmup),
        "ms_per_step": t / steps * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u1 (bit-packed)", "data": "synthetic",
        "config": {"workload": f"BASELINE config 5: {n}x{n} random mask (density 0.5) in "
                               f"{ws} row band(s): near^4 + volume + reach (target density "
                               f"0.05) + ccl::label (64-bit labels)",
                   "rows_per_rank": r1 - r0,
                   "exchange": "near^4: 4 packed rows each way per neighbour (NCCL send/recv);"
                               " volume: 8 B all-reduce; reach/ccl: border records "
                               "all-gathered (NCCL), device union-find",
                   "labelling": "reach and ccl::label of the mask share one band "
                                "union-find (reach_ccl_banded)",
                   "timing": "CUDA events on the bands' stream around the K steps "
                             "(exchanges included), max over ranks",
                   "l2": "no flush: each step's working set (mask, target, 64-bit labels) "
                         "exceeds L2"},
        "near4_volume": vol,
        "gpu_launches": dev.launches - l0, "clocks": clocks.summary()}


def fig3_result(args, dev, stream, local, n=7680):
    """The paper's Fig. 3 workload (specs/segmentation.imgql):
    grow(hI, vI) on a 7680x7680 blob-noise image.  The paper times it from
    "starting computation" to "saving file" (result on the host): ~600 ms on a
    TITAN Xp with VoxLogicA-GPU, 750-1100 ms with the CPU VoxLogicA.  Here: device
    time (input resident) and the paper's measure (host u16 in -> host mask out
    through the program API), plus the reference executor on the host cores."""
    import hashlib

    import torch

    from paper_2010_07284_b200 import PixelKind
    from paper_2010_07284_b200 import synth as S
    from paper_2010_07284_b200.executor import Program
    from paper_2010_07284_b200.imgql import STDLIB, compile_text

    spec = ('load img = "input.png"\nlet hI = intensity(img) >. 62258\n'
            'let vI = intensity(img) >. 56360\nlet gtv = grow(hI,vI)\n'
            'save "segmentation.png" gtv\n')
    img = S.blob_noise(n, n, 1)
    graph = compile_text(spec)
    prim = sum(1 for t in graph.nodes if t.opcode not in ("load", "save", "const"))
    out_task = [i for i, t in enumerate(graph.nodes) if t.opcode == "save"][0]
    prog = Program(graph, dev)
    pin_in = torch.from_numpy(img).pin_memory()
    pin_out = torch.empty((n, n), dtype=torch.uint8).pin_memory()
    prog.set_input_host("input.png", pin_in.numpy(), PixelKind.U16)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    for _ in range(3):
        prog.run()
    torch.cuda.synchronize()
    reps = max(3, min(args.steps, 10))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    for a, b in ev:
        flush.zero_()
        a.record(stream)
        prog.run()
        b.record(stream)
    torch.cuda.synchronize()
    ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    t0 = time.perf_counter()
    for _ in range(reps):
        prog.set_input_host("input.png", pin_in.numpy(), PixelKind.U16)
        prog.run()
        prog.download(out_task, pin_out.numpy())
    e2e_ms = (time.perf_counter() - t0) / reps * 1e3
    want = golden("fig3", "segmentation_sha256")
    ok = None
    if want:
        ok = hashlib.sha256(pin_out.numpy().tobytes()).hexdigest() == want
        assert ok, "Fig. 3 segmentation differs from the reference-pinned sha256"
    cpu = None
    if not args.no_cpu_baseline:
        import oracle as O
        if os.path.exists(O._REF):
            R = O.Reference(workers=os.cpu_count() or 1)
            res = R.run(spec, {"input.png": img}, STDLIB)
            cpu = {"value": prim * n * n / (res["computation_ms"] / 1e3) / 1e9,
                   "unit": "Gpixel-ops/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": "the whole spec through executor::run (computationMs, i.e. "
                             "'starting computation' to the end, saves included)",
                   "ms": res["computation_ms"]}
    return {"workload": f"Fig. 3: grow(hI, vI) on a {n}x{n} blob-noise image (seed 1), "
                        "specs/segmentation.imgql", "primitive_nodes": prim,
            "ms_device": ms, "value": prim * n * n / (ms / 1e3) / 1e9, "unit": "Gpixel-ops/s",
            "kernels_per_formula": prog.launches, "l2": "flushed before every timed step",
            "e2e": {"ms": e2e_ms, "value": prim * n * n / (e2e_ms / 1e3) / 1e9,
                    "unit": "Gpixel-ops/s", "h2d_bytes_per_step": n * n * 2,
                    "d2h_bytes_per_step": n * n,
                    "timing": "host wall clock: u16 H2D from pinned memory, program, "
                              "mask D2H (the paper's starting-computation-to-saved measure)"},
            "published": {"ms": 600, "hardware": "NVIDIA TITAN Xp (VoxLogicA-GPU, OpenCL)",
                          "source": "PAPER.md:463-481"},
            "speedup_vs_published_e2e": 600.0 / e2e_ms,
            "checksum_ok": ok, "cpu_baseline": cpu}


_GOLD = None


def golden(section, key):
    """Reference-pinned values (tests/golden/large_checksums.json, generated from the
    reference by tests/golden/make_golden_large.py) -- a committed data file."""
    global _GOLD
    if _GOLD is None:
        try:
            with open(os.path.join(ROOT, "tests", "golden", "large_checksums.json")) as f:
                _GOLD = json.load(f)
        except (OSError, ValueError):
            _GOLD = {}
    return _GOLD.get(section, {}).get(key)


def main():
    args = parse()
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference_arm(args, ws, rank)
        return
    if args.config != "c2":
        import torch

        from paper_2010_07284_b200 import Device
        torch.cuda.set_device(local)
        if ws > 1:
            init_dist(local)
        stream = torch.cuda.Stream(device=local)
        torch.cuda.set_stream(stream)
        dev = Device(local, stream=stream.cuda_stream)
        if args.config == "c4":
            line = c4_result(args, ws, rank, local, dev, stream,
                             n=args.size if args.size != 4096 else 16384)
        elif args.config == "c5":
            line = c5_result(args, ws, rank, local, dev, stream,
                             n=args.size if args.size != 4096 else 65536)
        else:
            line = formula_result(args, ws, rank, local, dev, stream, args.config)
        if rank == 0:
            print(json.dumps(line), flush=True)
        if ws > 1:
            torch.distributed.destroy_process_group()
        return

    import numpy as np
    import torch

    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        init_dist(local)
    from paper_2010_07284_b200 import (Device, DeviceImage, PixelKind, kernels, reach)
    from paper_2010_07284_b200 import synth as S
    from paper_2010_07284_b200.executor import Program
    from paper_2010_07284_b200.imgql import compile_text

    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    dev = Device(local, stream=stream.cuda_stream)

    size, depth = args.size, args.depth
    px = size * size
    img = S.blob_noise(size, size, args.seed)
    graph = compile_text(S.near_reach_chain(depth))
    prim_nodes = sum(1 for t in graph.nodes if t.opcode not in ("load", "save", "const"))
    out_task = [i for i, t in enumerate(graph.nodes) if t.opcode == "save"][0]
    prog = Program(graph, dev)
    pin_in = torch.from_numpy(img).pin_memory()
    pin_out = torch.empty((size, size), dtype=torch.uint8).pin_memory()
    prog.set_input_host("img.png", pin_in.numpy(), PixelKind.U16)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    cse = args.label_cse
    for _ in range(max(3, args.warmup)):
        prog.run(label_cse=cse)
    torch.cuda.synchronize()

    # ---- value: device-resident, per-step CUDA events, L2 flushed between steps
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches0 = dev.launches
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            prog.run(label_cse=cse)
            ends[i].record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    launches = dev.launches - launches0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_s = sum(step_ms) / 1e3
    if ws > 1:
        t = torch.tensor([total_s], device=f"cuda:{local}", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_s = float(t.item())
    value = ws * args.steps * prim_nodes * px / total_s / 1e9
    ms_per_step = total_s / args.steps * 1e3

    # secondary: the same formula with label CSE toggled (reported, not the headline)
    alt = None
    if args.alt_steps > 0:
        for _ in range(2):
            prog.run(label_cse=not cse)
        torch.cuda.synchronize()
        a_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(args.alt_steps)]
        for a0, a1 in a_ev:
            flush.zero_()
            a0.record(stream)
            prog.run(label_cse=not cse)
            a1.record(stream)
        torch.cuda.synchronize()
        alt_s = sum(a0.elapsed_time(a1) for a0, a1 in a_ev) / 1e3
        alt = {"label_cse": not cse, "value": args.steps and args.alt_steps * prim_nodes * px / alt_s / 1e9,
               "ms_per_step": alt_s / args.alt_steps * 1e3, "kernels_per_formula": prog.launches}
        prog.run(label_cse=cse)
        torch.cuda.synchronize()

    # correctness guard on the benchmarked output: the reference's own result of this
    # exact workload (executor::run, sha256 in tests/golden/large_checksums.json)
    import hashlib
    res = np.zeros((size, size), np.uint8)
    prog.download(out_task, res)
    checksum_ok = None
    want = (golden("c2", "sha256") or {}).get(f"x{depth}") if (size, args.seed) == (4096, 1) else None
    if want:
        checksum_ok = hashlib.sha256(res.tobytes()).hexdigest() == want
        assert checksum_ok, "C2 chain output differs from the reference-pinned sha256"

    # ---- e2e: host buffers through the public program API
    e2e = None
    if not args.no_e2e:
        for _ in range(2):
            prog.set_input_host("img.png", pin_in.numpy(), PixelKind.U16)
            prog.run(label_cse=cse)
            prog.download(out_task, pin_out.numpy())
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            prog.set_input_host("img.png", pin_in.numpy(), PixelKind.U16)
            prog.run(label_cse=cse)
            prog.download(out_task, pin_out.numpy())
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        if ws > 1:
            t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": ws * args.steps * prim_nodes * px / e2e_s / 1e9, "unit": "Gpixel-ops/s",
               "h2d_bytes_per_step": px * 2, "d2h_bytes_per_step": px,
               "ms_per_step": e2e_s / args.steps * 1e3, "timing": "host wall clock, synced"}
        assert np.array_equal(pin_out.numpy(), res)

    # ---- roofline of the dominant kernel.  With label CSE (default) that is
    # k_reach_chain: ONE persistent launch per formula running all 500 reaches; its
    # duration is read from a timeline run (CUDA events around every device step).
    # Without label CSE it is k_reach_fused, one launch per reach: duration = step
    # time / 500 (an upper bound: the ~10 us prologue is charged to the reaches).
    peak, peak_kind = measured_peak_gbs()
    n_reach = depth // 2
    chain_us = None
    if cse and n_reach > 0:
        durs = []
        for _ in range(3):
            prog.run(label_cse=cse, timeline=True)
            tt = prog.task_time(graph.nodes[out_task].deps[0])
            if tt:
                durs.append(tt[1] - tt[0])
        chain_us = statistics.median(durs) * 1e3 if durs else None
        prog.run(label_cse=cse)
        torch.cuda.synchronize()
    in_region = n_reach > 0 and not cse
    t_reach_region = ms_per_step / 1e3 / n_reach if in_region else None
    dimg = DeviceImage.upload(img, PixelKind.U16, dev)
    b = kernels.threshold(kernels.CmpOp.Gt, dimg, 56360, dev)
    t1 = kernels.dilate(kernels.threshold(kernels.CmpOp.Gt, dimg, 62258, dev), dev)
    reps = 20
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(reps)]
    ev_n = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(reps)]
    for _ in range(3):
        reach(t1, b, dev)
    torch.cuda.synchronize()
    for i in range(reps):
        flush.zero_()
        ev[i][0].record(stream)
        r = reach(t1, b, dev)
        ev[i][1].record(stream)
        flush.zero_()
        ev_n[i][0].record(stream)
        n = kernels.dilate(r, dev)
        ev_n[i][1].record(stream)
        del r, n
    torch.cuda.synchronize()
    t_reach = statistics.mean(a.elapsed_time(z) for a, z in ev) / 1e3
    t_near = statistics.mean(a.elapsed_time(z) for a, z in ev_n) / 1e3
    if chain_us:
        launch_s = chain_us / 1e6
        units = n_reach
        traffic, traffic_src = profiled_traffic("k_reach_chain")
        roofline = {
            "bound": "hbm", "kernel": "k_reach_chain (all 500 reaches of the chain in ONE "
                                      "persistent cooperative launch on a shared labelling of "
                                      "`through`; 64x256-px tiles, 7 per SM; per reach: "
                                      "staged window + stencils, sticky seed flags, an arrival "
                                      "(a tile waits only for the tiles that can still seed one "
                                      "of its shared roots), select, step-tagged halo records "
                                      "to the neighbouring tiles)",
            "achieved": BYTES_PER_PX["reach"] * px * units / launch_s / 1e9, "peak": peak,
            "unit": "GB/s",
            "frac": BYTES_PER_PX["reach"] * px * units / launch_s / 1e9 / peak,
            "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst)",
            "algorithmic_bytes_per_px": BYTES_PER_PX["reach"],
            "px_per_launch": px * units, "reaches_per_launch": units,
            "duration_us": chain_us, "share_of_step": chain_us / 1e3 / ms_per_step,
            "duration_source": "median of 3 timeline runs (CUDA events around the step)",
            "note": "frac >> 1 is not HBM evidence: SURVEY 8(d)'s 8.375 B/px per reach assume a "
                    "u32 labelling materialised per reach; here `through` is labelled once per "
                    "formula and every reach works on L2-resident bit images (DRAM `traffic` "
                    "per launch).  The kernel is bound by cross-SM latency: per reach the "
                    "neighbours' halo records (an L2 round trip) plus the window / seed / "
                    "select work of the slowest tiles; no grid barrier is paid",
            "latency_model": {
                "per_reach_us": chain_us / units,
                "grid_barrier_floor_us": 1.64,
                "barrier_source": "tools/ubench_barrier.cu, 592 co-resident CTAs "
                                  "(profiles/r02_ubench_barrier.txt)",
                "phase_timeline": "profiles/r02j_chain_phases.txt (SLCS_PHASE_TIMING=1)"},
            "compulsory_bytes_per_px": 0.375,
            "compulsory_frac": 0.375 * px * units / launch_s / 1e9 / peak,
        }
    else:
        if not in_region:
            t_reach_region = t_reach
        achieved = BYTES_PER_PX["reach"] * px / t_reach_region / 1e9
        traffic, traffic_src = profiled_traffic("k_reach_fused<1")
        roofline = {
            "bound": "hbm", "kernel": "k_reach_fused<0,64,2> (one cooperative launch per "
                                      "reach -- target near^2 from a staged window, tile-local "
                                      "run union-find, border unions, flag propagation, select; "
                                      "the closing near folds into the next reach)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": traffic_src,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}, burst)",
            "algorithmic_bytes_per_px": BYTES_PER_PX["reach"], "px_per_launch": px,
            "duration_us": t_reach_region * 1e6,
            "duration_source": (f"timed region / {n_reach} reach launches per step (CUDA "
                                "events)" if in_region else "standalone"),
            "note": "frac near or above 1: the 8.375 B/px of SURVEY 8(d) assume a materialised "
                    "u32 labelling; the fused kernel keeps labels in shared memory",
            "compulsory_bytes_per_px": 0.375,
            "compulsory_frac": 0.375 * px / t_reach_region / 1e9 / peak,
        }
    roofline["standalone_cold"] = {
        "kernel": "k_reach_fused<1,64,0> via reach() (one reach, L2 flushed)",
        "reach_ms": t_reach * 1e3, "achieved": BYTES_PER_PX["reach"] * px / t_reach / 1e9,
        "frac": BYTES_PER_PX["reach"] * px / t_reach / 1e9 / peak, "near_ms": t_near * 1e3,
        "near_achieved_gbs": BYTES_PER_PX["near"] * px / t_near / 1e9}

    prims = prims5 = None
    if rank == 0 and ws == 1 and not args.no_primitives:
        prims = primitive_table(dev, stream, local)
        prims5 = primitive_table(dev, stream, local, n=65536, reps=5, copies=2, labels=False)

    # the other BASELINE workloads: at N=1 all of them; at N>1 the two that shard
    # (C3 slices over ranks, C5 row bands), every rank taking part
    extra = {}
    if not args.no_extra:
        def guarded(fn, *a, **kw):
            # a failing sub-result is reported in the line, never fatal to the headline
            try:
                return fn(*a, **kw)
            except Exception as e:  # noqa: BLE001
                import traceback
                traceback.print_exc()
                return {"error": f"{type(e).__name__}: {e}"[:500]}
        extra["segmentation_c3"] = guarded(formula_result, args, ws, rank, local, dev, stream,
                                           "c3")
        extra["bands_c5"] = guarded(c5_result, args, ws, rank, local, dev, stream,
                                    n=args.c5_size)
        if ws == 1:
            extra["ccl_reach_c4"] = guarded(c4_result, args, ws, rank, local, dev, stream)
            extra["fig3_grow_7680"] = guarded(fig3_result, args, dev, stream, local)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            r = cpu_reference_sample(size, args.seed, args.ref_depth, 1)
            t = sum(r["times"])
            cpu = {"value": r["nodes"] * r["px"] / t / 1e9, "unit": "Gpixel-ops/s",
                   "cores": r["cores"], "kind": r["kind"], "sample": r["sample"],
                   "ms_per_formula_extrapolated": t / r["nodes"] * (depth + 2) * 1e3}
        except Exception as e:  # baseline is reported, never required
            cpu = {"value": None, "unit": "Gpixel-ops/s", "cores": os.cpu_count(),
                   "kind": "unavailable", "sample": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": "Gpixel-ops/s", "value": value, "unit": "Gpixel-ops/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "u1/u16 (bit-packed integer)", "data": "synthetic",
            "config": {"workload": f"BASELINE config 2: {depth}-deep near/reach chain on a "
                                   f"{size}x{size} blob-noise image (seed {args.seed})",
                       "image": f"{size}x{size}", "depth": depth, "tasks": graph.node_count(),
                       "primitive_nodes": prim_nodes, "l2": "flushed (512 MiB write) "
                                                              "before every timed step",
                       "parallelism": "replicas" if ws > 1 else "single",
                       "ms_per_formula": ms_per_step},
            "gpu_launches": launches, "kernels_per_formula": prog.launches,
            "label_cse": cse, "alternate": alt, "checksum_ok": checksum_ok,
            "clocks": clocks.summary(), "e2e": e2e, "roofline": roofline,
            "cpu_baseline": cpu, **extra, "primitives_c4": prims, "primitives_c5": prims5,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
