"""The reference CPU path at full length, once (SURVEY.md §8(d) "CPU path timed beside it").

Runs the unmodified reference (oracle/_ref, Release -O3) on this host's cores and prints
one JSON object:
  * C2 (ii): the near/reach chain at 4096^2 through `executor::run` at depths 10 and 20
    (the linear fit of acceptance criterion 9) and, with --full, at depth 1000;
  * C4: `ccl::label` and `reach` on the 16384^2 random mask (density 0.5, Rng seed 1;
    target density 0.05, seed 2), timed around the direct calls.
Test/measurement infrastructure: this is the CPU baseline, not the product.

  python tools/cpu_reference_runs.py [--full] [--out profiles/r01f_cpu_reference.json]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--full", action="store_true", help="also run the depth-1000 chain")
    p.add_argument("--c4-size", type=int, default=16384)
    p.add_argument("--out", default=None)
    a = p.parse_args()

    import oracle as O
    from paper_2010_07284_b200 import synth as S
    from paper_2010_07284_b200.imgql import STDLIB

    if not O.ref_available():
        sys.exit("oracle/_ref is not built")
    cores = os.cpu_count() or 1
    R = O.Reference(workers=cores)
    out = {"cores": cores, "build": "oracle/_ref (reference sources, -O3 -DNDEBUG)"}

    img = S.blob_noise(4096, 4096, 1)
    chain = {}
    for depth in (10, 20) + ((1000,) if a.full else ()):
        res = R.run(S.near_reach_chain(depth), {"img.png": img}, STDLIB)
        ms = res["computation_ms"]
        chain[str(depth)] = {"computation_ms": ms, "primitive_nodes": depth + 2,
                             "gpixel_ops_per_s": (depth + 2) * 4096 * 4096 / ms / 1e6}
        print(f"chain depth {depth}: {ms / 1e3:.2f} s", file=sys.stderr, flush=True)
    d10, d20 = chain["10"]["computation_ms"], chain["20"]["computation_ms"]
    slope = (d20 - d10) / 10
    chain["linear_fit"] = {"ms_per_step": slope, "intercept_ms": d10 - 10 * slope,
                           "depth_1000_ms": d10 + 990 * slope}
    out["c2_chain_4096"] = chain

    n = a.c4_size
    mask = O.random_mask(n, n, 0.5, O.Rng(1))
    target = O.random_mask(n, n, 0.05, O.Rng(2))
    t0 = time.perf_counter()
    R.ccl_label(mask)
    t_ccl = time.perf_counter() - t0
    print(f"c4 ccl: {t_ccl:.2f} s", file=sys.stderr, flush=True)
    t0 = time.perf_counter()
    R.reach(target, mask)
    t_reach = time.perf_counter() - t0
    print(f"c4 reach: {t_reach:.2f} s", file=sys.stderr, flush=True)
    out["c4_random_0.5"] = {"size": n, "ccl_label_s": t_ccl, "reach_s": t_reach,
                            "gpixel_ops_per_s": 2 * n * n / (t_ccl + t_reach) / 1e9}
    text = json.dumps(out, indent=1)
    print(text)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text + "\n")


if __name__ == "__main__":
    main()
