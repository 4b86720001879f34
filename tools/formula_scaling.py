"""Large-formula scaling (the paper's §4.1 experiment; the reference's `bench`
subcommand, proj/src/bench.cpp:18-85) on the device program path.

For each formula size: generate the input (blob noise, synth.cpp:43-81) and the
formula (`sequential` = gen::sequentialFormula, formula_gen.cpp:8-17; `chain` =
the config-2 near/reach chain), compile once, run `--warmup` untimed and
`--reps` timed evaluations (CUDA events around each device-resident run), and
print the reference's CSV (bench.cpp:66-75):

  kind,size,seed,workers,tasks,wall_ms_mean,wall_ms_stddev

`workers` is 0: the device has no worker pool.  `--gnuplot FILE` writes the
reference's plot script (bench.cpp:77-85).

  python tools/formula_scaling.py --kind chain --sizes 10,100,1000 --image 4096
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--kind", choices=["sequential", "chain"], default="chain")
    p.add_argument("--sizes", default="10,50,100,500,1000")
    p.add_argument("--image", type=int, default=4096)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=2)
    p.add_argument("--gnuplot", default=None)
    a = p.parse_args()

    import torch

    from paper_2010_07284_b200 import Device, PixelKind
    from paper_2010_07284_b200 import synth as S
    from paper_2010_07284_b200.executor import Program
    from paper_2010_07284_b200.imgql import compile_text

    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    dev = Device(0, stream=stream.cuda_stream)
    img = S.blob_noise(a.image, a.image, a.seed)
    print("kind,size,seed,workers,tasks,wall_ms_mean,wall_ms_stddev")
    for size in (int(x) for x in a.sizes.split(",")):
        if a.kind == "chain":
            text, name = S.near_reach_chain(size), "img.png"
            inp = img
        else:
            text, name = S.sequential_formula(size), "x.png"
            inp = (img > 56360).astype("uint8")
        graph = compile_text(text)
        prog = Program(graph, dev)
        prog.set_input_host(name, inp, PixelKind.U16 if a.kind == "chain" else PixelKind.Bool)
        for _ in range(a.warmup):
            prog.run(label_cse=False)
        torch.cuda.synchronize()
        times = []
        for _ in range(a.reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            prog.run(label_cse=False)
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
        sd = statistics.pstdev(times) if len(times) > 1 else 0.0
        print(f"{a.kind},{size},{a.seed},0,{graph.node_count()},{statistics.mean(times):.3f},"
              f"{sd:.3f}", flush=True)
    if a.gnuplot:
        with open(a.gnuplot, "w") as f:
            f.write("set datafile separator ','\nset key autotitle columnhead\n"
                    "set xlabel 'formula size'\nset ylabel 'wall ms'\n"
                    "plot 'scaling.csv' using 2:6 with linespoints title 'mean wall ms'\n")


if __name__ == "__main__":
    main()
