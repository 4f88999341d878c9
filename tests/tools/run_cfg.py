"""Developer harness (not the bench): time one BASELINE workload with a given
kernel configuration and print the per-phase split and the BCD sub-phases.
    python tests/tools/run_cfg.py --cfg C --r 12 --copies 8
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_1701_05363_b200 as somf_pkg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="C", choices=["B", "C", "D", "E"])
    ap.add_argument("--r", type=float, default=12.0)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--burn", type=int, default=20)
    ap.add_argument("--copies", type=int, default=0)
    ap.add_argument("--bcd-kernel", default="auto")
    ap.add_argument("--tile-rows", type=int, default=0)
    ap.add_argument("--group", type=int, default=0)
    ap.add_argument("--codes-kernel", default="auto")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    if args.cfg == "C":
        w = bench.WORKLOAD
        batches, d0 = bench.fmri_inputs_gpu(8, w["eta"], w["k"], 0, dev)
        p, k, eta = d0.shape[0], w["k"], w["eta"]
        kw = dict(lam=w["lam"], nu=w["nu"], mu=w["mu"])
    else:
        gen_cls, k, eta, kw = {
            "B": (bench.HyperspectralStreamGPU, 256, 256, dict(lam=0.1, nu=0.0, mu=1.0)),
            "D": (bench.NmfStreamGPU, 128, 512, dict(lam=0.05, nu=1.0, mu=1.0, pos_code=True, pos_dict=True)),
            "E": (bench.FmriEStreamGPU, 256, 512, dict(lam=0.05, nu=0.0, mu=0.5)),
        }[args.cfg]
        gen = gen_cls(eta, seed=0, device=dev)
        batches = [gen.batch() for _ in range(8)]
        d0 = gen.batch(k)
        p = gen.p
    m = somf_pkg.Somf(p, k, eta, r=args.r, u=0.917, seed=0, device=0, stream=stream, bcd_copies=args.copies,
                      bcd_kernel=args.bcd_kernel, bcd_tile_rows=args.tile_rows, codes_kernel=args.codes_kernel,
                      bcd_group=args.group, **kw)
    m.set_components(d0)
    for i in range(args.burn):
        m.partial_fit(batches[i % len(batches)])
    torch.cuda.synchronize()
    ms = bench.time_steps(m, batches, args.burn, args.steps, flush, stream)
    m.profile_read()
    m.profile_enable(True)
    bench.time_steps(m, batches, args.burn + args.steps, args.steps, flush, stream)
    pr = m.profile_read()
    cyc = m.bcd_phase_cycles()
    m.profile_enable(False)
    n = max(cyc["launches"], 1)
    mhz = 1965.0
    out = dict(cfg=args.cfg, r=args.r, p=p, k=k, eta=eta, ms_per_step=sum(ms) / len(ms), bcd=m.bcd_variant,
               kernels=m.last_kernels(), info=m.last_step_info(),
               phase_ms={ph: v / max(pr["steps"], 1) for ph, v in pr["ms"].items() if v > 0},
               bcd_us={ph: round(v / n / mhz, 2) for ph, v in cyc.items() if isinstance(v, int) and ph != "launches"},
               update_us={ph: round(v / n / mhz, 2) for ph, v in cyc["update_split"].items()},
               setup_us={ph: round(v / n / mhz, 2) for ph, v in cyc["setup_split"].items()},
               ridge_us={ph: round(v / n / mhz, 2) for ph, v in cyc["ridge"].items() if isinstance(v, int)},
               unconverged=[round(u / n, 1) for u in cyc["unconverged_per_round"] if u],
               cd=cyc["cd"],
               big_us={nm: round(cyc["raw"][i] / n / mhz, 2) for nm, i in
                       (("tile_load", 82), ("setup_stage", 83), ("setup_permute", 93), ("setup_r0", 94),
                        ("setup_radii_scratch", 95))})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
