"""Host executor: runs a TaskGraph as one device-resident program.

Mirrors ``executor::run`` (proj/src/executor.cpp:231-282, RunOptions /
RunReport at executor.hpp:16-50) but evaluates the whole DAG through
``slcs_program_*`` (csrc/program.cu): one fused, liveness-planned CUDA graph
instead of one CPU task per node.  ``load`` takes images supplied by the
caller or, with ``RunOptions.baseDir``, reads PNG files (png_io.cpp via
csrc/png.cu); ``save`` keeps the result on the device, exposes it by path and,
with ``baseDir``, writes the PNG.
"""
from __future__ import annotations

import ctypes as C
import os
import time
import math
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _lib
from .imgql import TaskGraph, compile_text
from .pixlog import (_DTYPE, Device, DeviceImage, ImageBuffer, PixelKind, RunError, _check,
                     loadPng, pixelKindName, savePng)

FLAG_GRAPH = 1
FLAG_NO_FUSION = 2
FLAG_NO_LABEL_CSE = 4
FLAG_NO_CHAIN = 8
FLAG_TIMELINE = 16


def format_number(v: float) -> str:
    """formatNumber (image.cpp:64-68): snprintf "%.6g".  glibc prints a NaN with
    its sign bit set (e.g. inf - inf on x86) as "-nan"; Python's % prints "nan"
    for every NaN, so the sign is restored here."""
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.6g" % v


@dataclass
class RunOptions:
    device: Optional[Device] = None
    fusion: bool = True
    cuda_graph: bool = True
    label_cse: bool = True
    chain: bool = True
    # RunOptions::baseDir (executor.hpp:16-26): when set, `load` paths not supplied
    # in `images` are read as PNG from here and every `save` writes its PNG here
    baseDir: Optional[str] = None
    # per-task device timeline (events between the device steps, eager launches):
    # fills RunReport.events and logs "task <id> <opcode> <ms>ms" (executor.cpp:184-189)
    timeline: bool = False
    log: Optional[object] = None  # callable(line); RunOptions::log (executor.hpp:21-22)


@dataclass
class RunReport:
    computationMs: float = 0.0
    taskCount: int = 0
    printLines: list = field(default_factory=list)
    savedFiles: list = field(default_factory=list)
    outputs: dict = field(default_factory=dict)  # save path -> DeviceImage
    launches: int = 0
    plan: str = ""
    # TaskEvent per node (executor.hpp:28-35): id, opcode, ran, evaluations, startMs,
    # endMs (device time from the start of the run), and `step`: the device step
    # that evaluated it (a node fused into a consumer's launch reports that step)
    events: list = field(default_factory=list)


class Program:
    """A TaskGraph compiled for the device (slcs_program)."""

    def __init__(self, graph: TaskGraph, device: Optional[Device] = None):
        self.graph = graph
        self.device = device or Device.default()
        n = graph.node_count()
        ops = (C.c_char_p * max(1, n))(*[t.opcode.encode() for t in graph.nodes])
        nums = (C.c_double * max(1, n))(*[t.payload if isinstance(t.payload, float) else 0.0
                                          for t in graph.nodes])
        strs = (C.c_char_p * max(1, n))(*[t.payload.encode() if isinstance(t.payload, str)
                                          else None for t in graph.nodes])
        off = [0]
        deps: list[int] = []
        for t in graph.nodes:
            deps.extend(t.deps)
            off.append(len(deps))
        doff = (C.c_int * len(off))(*off)
        dd = (C.c_int * max(1, len(deps)))(*deps)
        h = C.c_void_p()
        _check(_lib.load().slcs_program_create(self.device.handle, n, ops, nums, strs, doff, dd,
                                               C.byref(h)))
        self.handle = h
        self.load_names = sorted({t.payload for t in graph.nodes if t.opcode == "load"})

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and _lib._lib is not None:
            _lib._lib.slcs_program_destroy(h)
            self.handle = None

    def bind(self, name: str, img: Union[ImageBuffer, DeviceImage, np.ndarray],
             kind: Optional[PixelKind] = None) -> None:
        if isinstance(img, ImageBuffer):
            self.set_input_host(name, img.data, img.kind())
            return
        if isinstance(img, np.ndarray):
            if kind is None:
                kind = PixelKind.U16 if img.dtype == np.uint16 else PixelKind.Bool
            self.set_input_host(name, img, kind)
            return
        _check(_lib.load().slcs_program_bind(self.handle, name.encode(), img.handle))

    def set_input_host(self, name: str, arr: np.ndarray, kind: PixelKind) -> None:
        a = np.ascontiguousarray(arr, _DTYPE[PixelKind(kind)])
        b, h, w = (1, *a.shape) if a.ndim == 2 else a.shape
        _check(_lib.load().slcs_program_set_input_host(self.handle, name.encode(), int(kind), w,
                                                       h, b, C.c_void_p(a.ctypes.data)))

    def run(self, fusion: bool = True, cuda_graph: bool = True, label_cse: bool = True,
            chain: bool = True, timeline: bool = False) -> None:
        flags = ((FLAG_GRAPH if cuda_graph else 0) | (0 if fusion else FLAG_NO_FUSION)
                 | (0 if label_cse else FLAG_NO_LABEL_CSE) | (0 if chain else FLAG_NO_CHAIN)
                 | (FLAG_TIMELINE if timeline else 0))
        _check(_lib.load().slcs_program_run(self.handle, flags))

    def result(self, task: int) -> Union[DeviceImage, float]:
        k, h, d = C.c_int(), C.c_void_p(), C.c_double()
        _check(_lib.load().slcs_program_result(self.handle, task, C.byref(k), C.byref(h),
                                               C.byref(d)))
        return d.value if k.value == 1 else DeviceImage(h, self.device)

    def download(self, task: int, out: Optional[np.ndarray] = None) -> Union[np.ndarray, float]:
        t = self.graph.nodes[task]
        res_kind = self.value_kind(task)
        if res_kind is None:
            d = C.c_double()
            _check(_lib.load().slcs_program_download(self.handle, task, C.byref(d), 8))
            return d.value
        if out is None:
            raise RunError("download of an image needs an output array", 7)
        _check(_lib.load().slcs_program_download(self.handle, task, C.c_void_p(out.ctypes.data),
                                                 out.nbytes))
        return out

    def task_time(self, task: int):
        """(start_ms, end_ms) of the device step that evaluated `task` in the last
        timeline run, or None."""
        a, b = C.c_float(), C.c_float()
        _check(_lib.load().slcs_program_task_time(self.handle, task, C.byref(a), C.byref(b)))
        return None if a.value < 0 else (a.value, b.value)

    def value_kind(self, task: int):
        k = C.c_int()
        _check(_lib.load().slcs_program_result(self.handle, task, C.byref(k), None, None))
        return None if k.value == 1 else True

    @property
    def launches(self) -> int:
        n = C.c_int()
        _check(_lib.load().slcs_program_launches(self.handle, C.byref(n)))
        return n.value

    @property
    def plan(self) -> str:
        return _lib.load().slcs_program_plan(self.handle).decode()


def run(graph: TaskGraph, images: dict, options: Optional[RunOptions] = None) -> RunReport:
    """Evaluates `graph`; `images` maps load paths to ImageBuffer/DeviceImage/ndarray."""
    options = options or RunOptions()
    prog = Program(graph, options.device)
    for name in prog.load_names:
        if name in images:
            prog.bind(name, images[name])
        elif options.baseDir is not None:
            prog.bind(name, loadPng(os.path.join(options.baseDir, name), prog.device))
    rep = RunReport(taskCount=graph.node_count())
    t0 = time.perf_counter()
    err: Optional[RunError] = None
    log = options.log or (lambda line: None)
    log("starting computation")
    try:
        prog.run(options.fusion, options.cuda_graph, options.label_cse, options.chain,
                 options.timeline)
    except RunError as e:
        err = e
    prog.device.synchronize()
    rep.computationMs = (time.perf_counter() - t0) * 1e3
    if options.timeline:
        rep.events = task_events(graph, prog, err)
        for ev in rep.events:
            if ev["ran"]:
                log(f"task {ev['id']} {ev['opcode']} {ev['endMs'] - ev['startMs']:.3f}ms")
    for out in graph.outputs:
        t = graph.nodes[out]
        try:
            v = prog.result(out)
        except RunError:
            continue
        if t.opcode == "save":
            rep.savedFiles.append(t.payload)
            rep.outputs[t.payload] = v
            if options.baseDir is not None:
                savePng(os.path.join(options.baseDir, t.payload), v, prog.device)
        else:
            if isinstance(v, DeviceImage):
                desc = f"image({v.width}x{v.height},{pixelKindName(v.kind)})"
            else:
                desc = format_number(v)
            rep.printLines.append(f"{t.payload}={desc}")
    rep.launches = prog.launches
    rep.plan = prog.plan
    if err is not None:
        raise err
    return rep


def task_events(graph: TaskGraph, prog: Program, err: Optional[RunError] = None) -> list:
    """TaskEvents (executor.hpp:28-35) from a timeline run.  A node without a device
    step of its own (fused into a consumer's launch -- near folded into a reach, a
    reach inside a chain, a threshold inside a listing) reports the step of the
    first consumer that has one; host-side nodes (const/load/save/print) report the
    interval of their producer."""
    n = graph.node_count()
    times = [prog.task_time(i) for i in range(n)]
    consumers = [[] for _ in range(n)]
    for i, t in enumerate(graph.nodes):
        for d in t.deps:
            consumers[d].append(i)
    step = list(times)
    for i in range(n - 1, -1, -1):  # fused into a later consumer's step
        if step[i] is None:
            later = [step[c] for c in consumers[i] if step[c] is not None]
            if later:
                step[i] = min(later)
    for i, t in enumerate(graph.nodes):  # host-side nodes: after their producer
        if step[i] is None and t.deps and step[t.deps[0]] is not None:
            step[i] = (step[t.deps[0]][1], step[t.deps[0]][1])
    failed = set()
    if err is not None:
        import re
        m = re.match(r"task (\d+) ", str(err))
        if m:
            failed.add(int(m.group(1)))
    events = []
    for i, t in enumerate(graph.nodes):
        aborted = any(d in failed for d in t.deps)
        if aborted:
            failed.add(i)
        s0, s1 = step[i] if step[i] is not None else (0.0, 0.0)
        events.append({"id": i, "opcode": t.opcode, "ran": not aborted,
                       "evaluations": 0 if aborted else 1, "startMs": s0, "endMs": s1,
                       "own_step": times[i] is not None})
    return events


def run_text(text: str, images: dict, options: Optional[RunOptions] = None) -> RunReport:
    return run(compile_text(text), images, options)
