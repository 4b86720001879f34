"""GPU: whole formulas through the device program vs the reference.

Mirrors proj/tests/test_executor.cpp (print format, CSE, U16 coercion,
failure propagation, intensity identity, stdlib pipelines) and checks random
ImgQL formulas against the reference's own executor::run (oracle/_ref) --
with fusion on/off and CUDA-graph on/off, the analogue of the reference's
worker-count invariance tests (test_executor.cpp:229-240).
"""
import numpy as np
import pytest

import oracle as O
from paper_2010_07284_b200 import ImageBuffer, PixelKind, RunError, mask
from paper_2010_07284_b200.executor import Program, RunOptions, run_text
from paper_2010_07284_b200.imgql import STDLIB, compile_text

pytestmark = pytest.mark.gpu

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not available")


def B(a):
    a = np.asarray(a, np.uint8)
    return ImageBuffer(a.shape[1], a.shape[0], PixelKind.Bool, a)


def out_of(rep, path):
    return rep.outputs[path].numpy()


def test_load_save_round_trips_pixels(dev):
    rng = O.Rng(61)
    img = np.array([rng.below(65536) for _ in range(13 * 9)], np.uint16).reshape(9, 13)
    rep = run_text('load x = "in.png"\nsave "out.png" x\n', {"in.png": img})
    assert rep.taskCount == 2 + 0 or rep.taskCount >= 2
    assert np.array_equal(out_of(rep, "out.png"), img)
    assert rep.savedFiles == ["out.png"]


def test_contradiction_is_all_false_and_near_evaluates_once(dev):
    rng = O.Rng(62)
    m = O.random_mask(16, 16, 0.5, rng)
    g = compile_text('load x = "m.png"\nsave "out.png" near(x) & !near(x)\n', with_stdlib=False)
    assert g.count_opcode("near") == 1
    rep = run_text('load x = "m.png"\nsave "out.png" near(x) & !near(x)\n', {"m.png": m})
    assert out_of(rep, "out.png").sum() == 0
    assert rep.plan.count(" near^") == 1


def test_print_formats(dev):
    m = mask("xx../xx../..../...x").data
    rep = run_text('load x = "m.png"\nprint "vol" volume(x)\nprint "ratio" 1 / 3\n'
                   'print "img" near(x)\n', {"m.png": m})
    assert rep.printLines == ["vol=5", "ratio=0.333333", "img=image(4x4,bool)"]


@pytest.mark.parametrize("graph", [True, False])
def test_adjacent_volumes_share_one_launch(dev, graph):
    """Adjacent volume steps of any shapes run as one k_volume_multi launch; every
    count (and arithmetic on them) equals the popcount, run after run (the
    accumulators reset themselves)."""
    shapes = [(37, 5), (1000, 333), (64, 64), (4097, 129), (1, 1), (31, 2000), (256, 256),
              (2, 3), (129, 65)]
    imgs = {f"m{i}.png": O.random_mask(w, h, 0.3 + 0.05 * i, O.Rng(70 + i)) for i, (w, h)
            in enumerate(shapes)}
    text = "".join(f'load x{i} = "m{i}.png"\n' for i in range(len(shapes)))
    text += "".join(f'print "v{i}" volume(x{i})\n' for i in range(len(shapes)))
    text += 'print "s" volume(x0) + volume(x3)\n'
    want = [int(np.asarray(imgs[f"m{i}.png"]).sum()) for i in range(len(shapes))]
    for _ in range(3):
        rep = run_text(text, imgs, RunOptions(cuda_graph=graph))
        assert rep.printLines[:len(shapes)] == [f"v{i}={w}" for i, w in enumerate(want)]
        assert rep.printLines[-1] == f"s={want[0] + want[3]}"
    assert "[launch group lead]" in rep.plan and "volume" in rep.plan


def test_failure_propagation_keeps_independent_branches(dev):
    m = O.random_mask(8, 8, 0.5, O.Rng(1))
    with pytest.raises(RunError, match="cannot open file for reading"):
        run_text('load x = "m.png"\nload y = "absent.png"\nsave "good.png" near(x)\n'
                 'save "bad.png" near(y)\n', {"m.png": m})
    prog = Program(compile_text('load x = "m.png"\nload y = "absent.png"\n'
                                'save "good.png" near(x)\nsave "bad.png" near(y)\n'))
    prog.bind("m.png", m, PixelKind.Bool)
    with pytest.raises(RunError):
        prog.run()
    good = [i for i, t in enumerate(prog.graph.nodes) if t.payload == "good.png"][0]
    assert np.array_equal(prog.result(good).numpy(), O.dilate(m))


def test_division_by_zero_and_type_errors(dev):
    m = O.random_mask(8, 8, 0.5, O.Rng(2))
    with pytest.raises(RunError, match="division by zero"):
        run_text('print "q" 1 / 0\n', {})
    with pytest.raises(RunError, match="division by zero"):
        run_text('load x = "m.png"\nprint "q" 1 / (volume(x) - volume(x))\n', {"m.png": m})
    with pytest.raises(RunError, match="expects a numeric image, got bool"):
        run_text('load x = "m.png"\nsave "o.png" x >. 3\n', {"m.png": m})
    with pytest.raises(RunError, match="cannot save a number"):
        run_text('save "o.png" 3\n', {})


def test_intensity_is_identity(dev):
    img = np.array([O.Rng(64).below(65536) for _ in range(36)], np.uint16).reshape(6, 6)
    rep = run_text('load x = "in.png"\nsave "a.png" intensity(x)\n'
                   'save "b.png" intensity(intensity(x))\n', {"in.png": img})
    assert np.array_equal(out_of(rep, "a.png"), img)
    assert np.array_equal(out_of(rep, "b.png"), img)


def test_numeric_images_coerce_to_masks(dev):
    img = np.array([[0, 1, 40000, 0]], np.uint16)
    rep = run_text('load x = "in.png"\nprint "v" volume(x)\nsave "n.png" !x\n', {"in.png": img})
    assert rep.printLines[0] == "v=2"
    assert out_of(rep, "n.png").tolist() == [[1, 0, 0, 1]]


def test_threshold_with_a_computed_comparand(dev):
    rng = np.random.default_rng(5)
    img = rng.integers(0, 200, (40, 50), dtype=np.uint16)
    m = (img > 150).astype(np.uint8)
    rep = run_text('load i = "i.png"\nload m = "m.png"\nsave "o.png" i >. volume(m) / 10\n',
                   {"i.png": img, "m.png": m})
    assert np.array_equal(out_of(rep, "o.png"), O.threshold(0, img, m.sum() / 10))


@pytest.mark.parametrize("fusion", [True, False])
@pytest.mark.parametrize("graph", [True, False])
def test_stdlib_pipelines_vs_oracle(dev, fusion, graph):
    rng = O.Rng(65)
    a = O.random_mask(20, 20, 0.25, rng)
    b = O.random_mask(20, 20, 0.35, rng)
    opts = RunOptions(fusion=fusion, cuda_graph=graph)
    for expr, ref in [("grow(a,b)", O.grow(a, b)), ("surrounded(a,b)", O.surrounded(a, b)),
                      ("near(a) | interior(b)", O.logical_or(O.dilate(a), O.interior(b))),
                      ("touch(a,b)", O.touch(a, b)), ("reach(a,b)", O.reach(a, b)),
                      ("maxvol(a | b)", O.maxvol(O.logical_or(a, b)))]:
        rep = run_text(f'load a = "a.png"\nload b = "b.png"\nsave "o.png" {expr}\n',
                       {"a.png": a, "b.png": b}, opts)
        assert np.array_equal(out_of(rep, "o.png"), ref), expr


def test_segmentation_spec_vs_reference_golden(dev):
    import json
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    G = np.load(os.path.join(here, "golden", "reference_vectors.npz"))
    D = json.load(open(os.path.join(here, "golden", "reference_dags.json")))
    rep = run_text(D["specs"]["segmentation"], {"input.png": G["seg_in"]})
    assert np.array_equal(out_of(rep, "segmentation.png"), G["seg_out"])
    rep = run_text(D["specs"]["c1"], {"img.png": G["seg_in"]})
    assert np.array_equal(out_of(rep, "out.png"), G["c1_out"])


def test_sequential_chain_fuses_to_stencils(dev):
    # formula_gen.cpp:8-17: near / ! alternation; near(!e) fuses to !interior(e)
    expr = "x"
    for i in range(40):
        expr = f"near({expr})" if i % 2 == 0 else f"!({expr})"
    m = O.random_mask(300, 200, 0.02, O.Rng(8))
    ref = m
    for i in range(40):
        ref = O.dilate(ref) if i % 2 == 0 else O.logical_not(ref)
    for fusion in (True, False):
        rep = run_text(f'load x = "m.png"\nsave "o.png" {expr}\n', {"m.png": m},
                       RunOptions(fusion=fusion))
        assert np.array_equal(out_of(rep, "o.png"), ref)
        if fusion:
            assert rep.launches <= 22, rep.plan


def test_near_reach_chain_small(dev):
    img = O.blob_noise(256, 256, 1)
    b = O.threshold(0, img, 56360)
    x = O.threshold(0, img, 62258)
    lines = ['load img = "img.png"', "let b = img >. 56360", "let x0 = img >. 62258"]
    for k in range(10):
        lines.append(f"let x{2 * k + 1} = near(x{2 * k})")
        lines.append(f"let x{2 * k + 2} = reach(x{2 * k + 1}, b)")
        x = O.reach(O.dilate(x), b)
    lines.append('save "o.png" x20')
    rep = run_text("\n".join(lines) + "\n", {"img.png": img})
    assert np.array_equal(out_of(rep, "o.png"), x)


@pytest.mark.parametrize("thr", [45875, 52428, 58982])
def test_reach_chain_many_components_per_tile(dev, thr):
    """A random `through` of density 0.3 / 0.2 / 0.1 puts more distinct components in a
    chain tile than it has local ids (CH_MAXL): those runs take the global-root
    path and the tile waits on the global arrival count.  Exact vs the oracle."""
    from paper_2010_07284_b200 import synth as S
    w, h, depth = 2048, 1024, 8
    rng = np.random.default_rng(thr)
    img = rng.integers(0, 65536, size=(h, w), dtype=np.uint16)
    graph = compile_text(S.near_reach_chain(depth, through_thr=thr, target_thr=65000))
    out_task = [i for i, t in enumerate(graph.nodes) if t.opcode == "save"][0]
    prog = Program(graph, dev)
    prog.set_input_host("img.png", img, PixelKind.U16)
    prog.run()
    assert "chain of" in prog.plan, prog.plan
    out = np.zeros((h, w), np.uint8)
    prog.download(out_task, out)
    b, x = O.threshold(0, img, thr), O.threshold(0, img, 65000)
    for k in range(depth):
        x = O.dilate(x) if k % 2 == 0 else O.reach(x, b)
    assert np.array_equal(out, x)


@pytest.mark.parametrize("cse", [True, False])
@pytest.mark.parametrize("graph", [True, False])
def test_near_reach_chain_large_path_label_cse(dev, cse, graph):
    # > 256 px: the tiled path; the 6 reaches share `b`, so with label CSE on
    # the labelling of b is computed once per run (generation-stamped flags)
    img = O.blob_noise(700, 530, 5)
    b = O.threshold(0, img, 56360)
    x = O.threshold(0, img, 62258)
    lines = ['load img = "img.png"', "let b = img >. 56360", "let x0 = img >. 62258"]
    for k in range(6):
        lines.append(f"let x{2 * k + 1} = near(x{2 * k})")
        lines.append(f"let x{2 * k + 2} = reach(x{2 * k + 1}, b)")
        x = O.reach(O.dilate(x), b)
    lines.append('save "o.png" x12')
    prog = Program(compile_text("\n".join(lines) + "\n"))
    prog.set_input_host("img.png", img, PixelKind.U16)
    out = [i for i, t in enumerate(prog.graph.nodes) if t.opcode == "save"][0]
    for _ in range(3):  # replays must not see stale flag stamps
        prog.run(cuda_graph=graph, label_cse=cse)
        got = np.zeros(img.shape, np.uint8)
        prog.download(out, got)
        assert np.array_equal(got, x)
    assert ("shared labelling" in prog.plan) == cse


def random_formula(rng, budget):
    if budget <= 1:
        img = "imgA" if rng.below(2) else "imgB"
        cmp = [">.", ">=.", "<.", "<=."][rng.below(4)]
        return f"{img} {cmp} {rng.below(65536)}"
    k = rng.below(7 if budget >= 3 else 3)
    if k == 0:
        return f"!({random_formula(rng, budget - 1)})"
    if k in (1, 2):
        return f"near({random_formula(rng, budget - 1)})"
    left = 1 + rng.below(budget - 2)
    l, r = random_formula(rng, left), random_formula(rng, budget - 1 - left)
    if k == 3:
        return f"({l}) & ({r})"
    if k == 4:
        return f"({l}) | ({r})"
    if k == 5:
        return f"reach({l}, {r})"
    return f"surrounded({l}, {r})"


@needs_ref
@pytest.mark.parametrize("size", [(37, 29), (256, 256), (300, 280)])
def test_random_formulas_vs_reference_executor(dev, size):
    R = O.Reference(workers=2)
    w, h = size
    rng = O.Rng(1000 + w)
    imgA = O.blob_noise(w, h, 11)
    imgB = np.array([rng.below(65536) for _ in range(w * h)], np.uint16).reshape(h, w)
    for i in range(12):
        f = random_formula(rng, 3 + rng.below(10))
        spec = f'load imgA = "a.png"\nload imgB = "b.png"\nsave "o.png" {f}\n'
        want = R.run(spec, {"a.png": imgA, "b.png": imgB}, STDLIB, ["o.png"])["outputs"]["o.png"]
        for fusion in (True, False):
            rep = run_text(spec, {"a.png": imgA, "b.png": imgB}, RunOptions(fusion=fusion))
            assert np.array_equal(out_of(rep, "o.png"), want), (i, f, fusion)


def test_program_rerun_with_new_inputs(dev):
    prog = Program(compile_text('load a = "a.png"\nload b = "b.png"\nsave "o.png" grow(a, b)\n'))
    out = [i for i, t in enumerate(prog.graph.nodes) if t.opcode == "save"][0]
    rng = O.Rng(3)
    for _ in range(4):
        a = O.random_mask(200, 150, 0.1, rng)
        b = O.random_mask(200, 150, 0.45, rng)
        prog.set_input_host("a.png", a, PixelKind.Bool)
        prog.set_input_host("b.png", b, PixelKind.Bool)
        prog.run()
        got = np.zeros((150, 200), np.uint8)
        prog.download(out, got)
        assert np.array_equal(got, O.grow(a, b))


def test_batched_program(dev):
    # C3-shaped: a stack of slices evaluated as one batched program
    imgs = np.stack([O.blob_noise(240, 240, s) for s in range(100, 106)])
    spec = ('load img = "s.png"\nlet hI = intensity(img) >. 62258\n'
            'let vI = intensity(img) >. 56360\n'
            'save "o.png" maxvol(grow(hI, vI)) | surrounded(hI, vI)\n')
    rep = run_text(spec, {"s.png": imgs})
    got = out_of(rep, "o.png")
    for s in range(6):
        hI = O.threshold(0, imgs[s], 62258)
        vI = O.threshold(0, imgs[s], 56360)
        ref = O.logical_or(O.maxvol(O.grow(hI, vI)), O.surrounded(hI, vI))
        assert np.array_equal(got[s], ref), s


@pytest.mark.parametrize("k", [0, 1, 2, 3, 5])
def test_reach_closing_radius_absorbs_following_nears(dev, k):
    # reach followed by k nears: the planner folds them into the reach's closing
    # near (k_out = k + 1; the fused kernel handles k_out <= 4, larger radii
    # fall back to a separate stencil) -- every variant must equal the oracle
    img = O.blob_noise(1200, 900, 11)
    t = O.threshold(0, img, 62258)
    b = O.threshold(0, img, 56360)
    expr = "reach(t, b)"
    ref = O.reach(t, b)
    for _ in range(k):
        expr = f"near({expr})"
        ref = O.dilate(ref)
    rep = run_text(f'load t = "t.png"\nload b = "b.png"\nsave "o.png" {expr}\n',
                   {"t.png": t, "b.png": b})
    assert np.array_equal(out_of(rep, "o.png"), ref)


CHAIN_SHAPES = [
    "near(reach(near(near(a)), b))",                      # target near^2 folded, closing near^2
    "reach(reach(a, b), b)",                              # selection emitted, consumer tk = 1
    "near(reach(reach(near(a), b), b))",                  # tk 1 -> selection -> tk 1, k_out 2
    "reach(near(reach(near(reach(a, b)), b)), b)",        # tk 2 twice
    "reach(near(near(near(a))), b)",                      # tk 3: beyond the fused window
    "reach(reach(a, b), reach(a, b))",                    # shared reach: no selection emit
    "near(reach(a, b)) | reach(near(a), b)",              # two consumers of near(a)
    # a reach with a closing near (k_out >= 1, three grid barriers) launched right
    # before another reach on the same `through` (early launch of the second)
    "reach(reach(a, b), b) | reach(a, b)",
    "near(reach(reach(a, b), b)) & near(reach(a, b))",
    "reach(reach(reach(a, b), b) | a, b)",
]


@needs_ref
@pytest.mark.parametrize("shape", CHAIN_SHAPES)
@pytest.mark.parametrize("cse", [False, True])
def test_reach_folding_shapes_vs_reference_executor(dev, shape, cse):
    # the planner's reach/near folds (tk, emitted selections, closing radii) on the
    # fused cooperative kernel, checked against the reference's own executor
    R = O.Reference(workers=4)
    img = O.blob_noise(700, 500, 21)
    spec = ('load img = "img.png"\nlet a = img >. 62258\nlet b = img >. 56360\n'
            f'save "o.png" {shape}\n')
    want = R.run(spec, {"img.png": img}, STDLIB, ["o.png"])["outputs"]["o.png"]
    prog = Program(compile_text(spec))
    prog.set_input_host("img.png", img, PixelKind.U16)
    out = [i for i, t in enumerate(prog.graph.nodes) if t.opcode == "save"][0]
    for graph in (True, False):
        prog.run(cuda_graph=graph, label_cse=cse)
        got = np.zeros(img.shape, np.uint8)
        prog.download(out, got)
        assert np.array_equal(got, want), (shape, cse, graph, prog.plan)


@needs_ref
def test_random_formulas_vs_reference_executor_large(dev):
    # the fused/folded paths on random nestings at a size above the small-image path
    R = O.Reference(workers=4)
    w, h = 640, 480
    rng = O.Rng(4242)
    imgA = O.blob_noise(w, h, 13)
    imgB = O.blob_noise(w, h, 17)
    for i in range(8):
        f = random_formula(rng, 4 + rng.below(8))
        spec = f'load imgA = "a.png"\nload imgB = "b.png"\nsave "o.png" {f}\n'
        want = R.run(spec, {"a.png": imgA, "b.png": imgB}, STDLIB, ["o.png"])["outputs"]["o.png"]
        rep = run_text(spec, {"a.png": imgA, "b.png": imgB}, RunOptions())
        assert np.array_equal(out_of(rep, "o.png"), want), (i, f)


@pytest.mark.parametrize("w,h", [(200, 150), (700, 500)])
def test_components_opcode_labels_and_errors(dev, w, h):
    # components(x) (new, like maxvol): the canonical ccl::label image of a mask
    img = O.blob_noise(w, h, 9)
    a = O.threshold(0, img, 40000)
    rep = run_text('load img = "img.png"\nlet c = components(img >. 40000)\n'
                   'save "c.png" c\nprint "lab" c\n', {"img.png": img})
    assert np.array_equal(rep.outputs["c.png"].numpy(), O.flood_fill_label(a))
    assert rep.printLines == [f"lab=image({w}x{h},label)"]
    with pytest.raises(RunError, match="expects a boolean image, got label"):
        run_text('load img = "img.png"\nsave "o.png" near(components(img >. 1))\n',
                 {"img.png": img})


def test_components_saved_as_label_colours(dev, tmp_path):
    from PIL import Image
    img = O.blob_noise(96, 64, 2)
    Image.fromarray(img).save(tmp_path / "in.png")
    run_text('load img = "in.png"\nsave "lab.png" components(img >. 45000)\n', {},
             RunOptions(baseDir=str(tmp_path)))
    lab = O.flood_fill_label(O.threshold(0, img, 45000))
    want = np.array([[O.label_color(int(x)) for x in row] for row in lab], np.uint8)
    assert np.array_equal(np.array(Image.open(tmp_path / "lab.png").convert("RGB")), want)


@pytest.mark.parametrize("fusion", [True, False])
def test_small_maxvol_prologue_epilogue_folds(dev, fusion):
    # the planner folds a bool-only operand listing (prologue) and a bool-only
    # consumer listing (epilogue) into the small-image maxvol launch, and batches
    # independent small reaches; results must not depend on it
    rng = O.Rng(77)
    n_sl, h, w = 5, 61, 97
    a = np.stack([O.random_mask(w, h, 0.45, rng) for _ in range(n_sl)])
    b = np.stack([O.random_mask(w, h, 0.3, rng) for _ in range(n_sl)])
    cases = [
        ("maxvol(a & !b) | b", lambda x, y: O.logical_or(O.maxvol(O.logical_and(x, O.logical_not(y))), y)),
        ("!maxvol(a | b) & a", lambda x, y: O.logical_and(O.logical_not(O.maxvol(O.logical_or(x, y))), x)),
        ("maxvol(maxvol(a) | b)", lambda x, y: O.maxvol(O.logical_or(O.maxvol(x), y))),
        ("maxvol(a) | maxvol(b)", lambda x, y: O.logical_or(O.maxvol(x), O.maxvol(y))),
        ("reach(a, b) | reach(b, a)", lambda x, y: O.logical_or(O.reach(x, y), O.reach(y, x))),
    ]
    for expr, ref in cases:
        prog = Program(compile_text(f'load a = "a.png"\nload b = "b.png"\nsave "o.png" {expr}\n'))
        prog.bind("a.png", a, PixelKind.Bool)
        prog.bind("b.png", b, PixelKind.Bool)
        prog.run(fusion=fusion)
        got = np.zeros((n_sl, h, w), np.uint8)
        prog.download(prog.graph.outputs[0], got)
        for s in range(n_sl):
            assert np.array_equal(got[s], ref(a[s], b[s])), (expr, s, prog.plan)


@needs_ref
def test_nan_and_inf_prints_match_reference_executor(dev):
    """print of NaN/inf results reads like the reference's snprintf("%.6g")
    (image.cpp:64-68): an invalid operation on x86 gives a NaN with the sign bit
    set ("-nan"), a propagated NaN keeps its operand's sign; the device
    arithmetic reproduces both (program.cu k_arith)."""
    R = O.Reference(workers=1)
    m = mask("x...\n.x..\n..x.\n...x")
    img = np.asarray(m.data, np.uint8)
    spec = ('load x = "m.png"\n'
            'print "a" 1e400 - 1e400\n'
            'print "b" (volume(x) * 1e400) - 1e400\n'
            'print "c" 0 * (volume(x) * 1e400)\n'
            'print "d" ((volume(x) * 1e400) - 1e400) * (0 - 1)\n'
            'print "e" (0 - 1) * 1e400 + volume(x)\n'
            'print "f" volume(x) / 3\n')
    want = R.run(spec, {"m.png": img}, STDLIB)["prints"]
    rep = run_text(spec, {"m.png": B(img)})
    assert rep.printLines == want


@pytest.mark.parametrize("nears,tail", [(0, 1), (2, 3), (1, 2), (2, 0)])
def test_reach_chain_radii(dev, nears, tail):
    """Chains whose reaches are separated by 0, 1 or 2 nears (the chain kernel's
    kmid) and end with 0..3 closing nears (klast), against the oracle."""
    w, h, n = 1500, 900, 7
    img = O.blob_noise(w, h, 17)
    lines = ['load img = "img.png"', "let b = img >. 56360", "let x0 = img >. 62258"]
    for k in range(n):
        t = f"x{k}"
        for _ in range(nears):
            t = f"near({t})"
        lines.append(f"let x{k + 1} = reach({t}, b)")
    res = f"x{n}"
    for _ in range(tail):
        res = f"near({res})"
    lines.append(f'save "out.png" {res}')
    graph = compile_text("\n".join(lines) + "\n")
    out_task = [i for i, t in enumerate(graph.nodes) if t.opcode == "save"][0]
    prog = Program(graph, dev)
    prog.set_input_host("img.png", img, PixelKind.U16)
    prog.run()
    out = np.zeros((h, w), np.uint8)
    prog.download(out_task, out)
    b, x = O.threshold(0, img, 56360), O.threshold(0, img, 62258)
    for _ in range(n):
        for _ in range(nears):
            x = O.dilate(x)
        x = O.reach(x, b)
    for _ in range(tail):
        x = O.dilate(x)
    assert np.array_equal(out, x), prog.plan


@pytest.mark.parametrize("w,h,depth", [(700, 500, 20), (1000, 1001, 12), (4100, 37, 9),
                                       (300, 2600, 30), (2048, 2048, 41)])
def test_reach_chain_one_launch_matches_oracle(dev, w, h, depth):
    """The config-2 chain with label CSE runs its reaches as ONE persistent launch
    (k_reach_chain); results equal the unchained label-CSE path, the per-reach
    fused path, and the CPU oracle of the same chain."""
    from paper_2010_07284_b200 import synth as S
    img = O.blob_noise(w, h, 5)
    graph = compile_text(S.near_reach_chain(depth))
    out_task = [i for i, t in enumerate(graph.nodes) if t.opcode == "save"][0]
    res = {}
    for name, kw in {"chain": {}, "cse": {"chain": False}, "fused": {"label_cse": False}}.items():
        prog = Program(graph, dev)
        prog.set_input_host("img.png", img, PixelKind.U16)
        for _ in range(2):
            prog.run(**kw)
        out = np.zeros((h, w), np.uint8)
        prog.download(out_task, out)
        res[name] = out
        if name == "chain":
            assert "chain of" in prog.plan, prog.plan
    b = O.threshold(0, img, 56360)
    x = O.threshold(0, img, 62258)
    for k in range(depth):
        x = O.dilate(x) if k % 2 == 0 else O.reach(x, b)
    assert np.array_equal(res["chain"], x)
    assert np.array_equal(res["cse"], x)
    assert np.array_equal(res["fused"], x)


def test_timeline_task_events_respect_dependencies(dev):
    """RunOptions.timeline fills RunReport.events like the reference's TaskEvents
    (executor.hpp:28-35, tests/test_executor.cpp "events respect the dependency
    partial order") and logs "task <id> <opcode> <ms>ms" lines."""
    from paper_2010_07284_b200 import synth as S
    img = O.blob_noise(700, 500, 3)
    lines = []
    graph = compile_text(S.near_reach_chain(8) + 'print "v" volume(x8)\n')
    rep = run_text(S.near_reach_chain(8) + 'print "v" volume(x8)\n', {"img.png": img},
                   RunOptions(timeline=True, log=lines.append))
    assert lines[0] == "starting computation"
    assert len(rep.events) == graph.node_count()
    for ev in rep.events:
        assert ev["evaluations"] == 1 and ev["ran"]
        assert ev["endMs"] >= ev["startMs"] >= 0
        for d in graph.nodes[ev["id"]].deps:
            assert ev["startMs"] >= rep.events[d]["startMs"] - 1e-6
    assert any(ev["own_step"] and ev["endMs"] > ev["startMs"] for ev in rep.events)
    assert sum(1 for l in lines if l.startswith("task ")) == graph.node_count()
    # the timeline run computes the same results
    want = run_text(S.near_reach_chain(8), {"img.png": img}).outputs["out.png"].numpy()
    assert np.array_equal(rep.outputs["out.png"].numpy(), want)
