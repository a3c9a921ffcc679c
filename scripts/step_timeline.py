"""In-graph kernel timeline of decode steps (torch.profiler / CUPTI activity records of the graph
replays): per-kernel-class durations as they run inside the captured step, the sum of kernel time
against the step's wall time (the launch gaps), and the largest gaps with the kernels around them.

    python scripts/step_timeline.py [--steps 5] [--ctx 32768]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ctx", type=int, default=32768)
    ap.add_argument("--model", default="llama-3.1-8b")
    ap.add_argument("--out", default="gpurun_out/step_timeline.json")
    args = ap.parse_args()
    import torch
    from paper_2502_04077_b200.decode import SHAPES, DecodeEngine
    from paper_2502_04077_b200.selector import SelectorConfig

    shape = SHAPES[args.model]
    eng = DecodeEngine(shape, 1, args.ctx, max_new=64, cfg=SelectorConfig(budget=1024),
                       group=shape.n_q_heads // shape.n_kv_heads)
    eng.init_history()
    eng.step(use_graph=False)
    eng.capture_all()
    for _ in range(6):
        eng.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    variants = []
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(args.steps):
            variants.append(eng.step())
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    kern = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
    kern = [k for k in kern if "Memcpy" not in k[2] and "Memset" not in k[2]]
    if not kern:
        print("no kernel records (CUPTI did not trace the graph replays)")
        return
    t0, t1 = kern[0][0], max(k[1] for k in kern)
    busy, gaps, cls = 0.0, [], collections.defaultdict(list)
    last_end, last_name = kern[0][0], None
    for s, e, n in kern:
        short = n.split("(")[0].replace("void ", "")[:60]
        cls[short].append(e - s)
        if s > last_end:
            gaps.append((s - last_end, last_name, short))
        busy += max(0.0, e - max(s, last_end))
        if e > last_end:
            last_end, last_name = e, short
    wall = t1 - t0
    # critical-path share: each kernel's end minus the previous kernel's end (launch order), so that
    # programmatic-dependent-launch overlap is charged to whoever finishes later
    inc = collections.defaultdict(float)
    inc_after = collections.defaultdict(list)  # (kernel, the kernel launched before it) -> critical shares
    prev_end, prev_name = t0, "-"
    for s_, e, n in sorted(kern, key=lambda x: x[0]):
        short = n.split("(")[0].replace("void ", "")[:60]
        d = max(0.0, e - prev_end)
        inc[short] += d
        inc_after[(short, prev_name)].append(d)
        prev_end, prev_name = max(prev_end, e), short
    out = {"steps": args.steps, "variants": variants, "wall_us_per_step": wall / args.steps,
           "kernel_busy_us_per_step": busy / args.steps, "gap_us_per_step": (wall - busy) / args.steps,
           "kernels_per_step": len(kern) / args.steps,
           "classes": {k: {"n_per_step": len(v) / args.steps, "mean_us": sum(v) / len(v),
                           "us_per_step": sum(v) / args.steps, "critical_us_per_step": inc[k] / args.steps}
                       for k, v in sorted(cls.items(), key=lambda kv: -sum(kv[1]))},
           "critical_by_predecessor": sorted(({"kernel": k, "after": a, "n_per_step": len(v) / args.steps,
                                              "mean_us": sum(v) / len(v)} for (k, a), v in inc_after.items()),
                                             key=lambda x: -x["mean_us"] * x["n_per_step"])[:16],
           "largest_gaps": [{"us": g, "after": a, "before": b} for g, a, b in sorted(gaps, reverse=True)[:12]]}
    n1 = len(kern) // args.steps  # the last step's raw records (start, end relative to its first kernel)
    last = kern[-n1:]
    out["last_step"] = [[round(s_ - last[0][0], 3), round(e - last[0][0], 3), n.split("(")[0].replace("void ", "")[:60]]
                        for s_, e, n in last]
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wall {out['wall_us_per_step']:.1f} us/step, kernels busy {out['kernel_busy_us_per_step']:.1f}, "
          f"gaps {out['gap_us_per_step']:.1f}, {out['kernels_per_step']:.0f} kernels/step")
    for k, v in list(out["classes"].items())[:14]:
        print(f"  {k:52s} {v['n_per_step']:5.1f}/step  mean {v['mean_us']:7.2f} us  {v['us_per_step']:7.1f} us/step"
              f"  critical {v['critical_us_per_step']:7.1f} us/step")
    print("critical share by predecessor:")
    for r in out["critical_by_predecessor"][:10]:
        print(f"  {r['kernel'][:44]:44s} after {r['after'][:44]:44s} {r['n_per_step']:5.1f}/step {r['mean_us']:7.2f} us")
    for g in out["largest_gaps"][:6]:
        print(f"  gap {g['us']:.2f} us  after {g['after']}  before {g['before']}")


if __name__ == "__main__":
    main()
