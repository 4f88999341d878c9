"""Developer harness: run a BASELINE workload step by step with every call
checked and report the first step whose BCD hits its round cap, with the
per-round unconverged-atom profile of that step.

    python tests/tools/cap_repro.py --cfg E --r 24 --steps 20
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
    ap.add_argument("--cfg", default="E", choices=["B", "D", "E"])
    ap.add_argument("--r", type=float, default=24.0)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--bcd-kernel", default="auto")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    gen_cls, k, eta, kw = {
        "B": (bench.HyperspectralStreamGPU, 256, 256, dict(lam=0.1, nu=0.0, mu=1.0)),
        "D": (bench.NmfStreamGPU, 128, 512, dict(lam=0.05, nu=1.0, mu=1.0, pos_code=True, pos_dict=True)),
        "E": (bench.FmriEStreamGPU, 256, 512, dict(lam=0.05, nu=0.0, mu=0.5)),
    }[args.cfg]
    gen = gen_cls(eta, seed=0, device=dev)
    pool = [gen.batch() for _ in range(8)]
    d0 = gen.batch(k)
    m = somf_pkg.Somf(gen.p, k, eta, r=args.r, u=0.917, seed=0, device=0, bcd_kernel=args.bcd_kernel, **kw)
    m.set_components(d0)
    m.profile_enable(True)
    for t in range(args.steps):
        m.bcd_phase_cycles()                # (each read resets the counters)
        m.partial_fit(pool[t % len(pool)])
        torch.cuda.synchronize()
        cyc = m.bcd_phase_cycles()
        unc = cyc["unconverged_per_round"]
        try:
            info = m.last_step_info()
            print(json.dumps({"cfg": args.cfg, "r": args.r, "t": t + 1, "ok": True, "q": info["q"],
                              "nred": info["bcd_reductions"], "bcd": m.bcd_variant,
                              "prefix_regressions": cyc["raw"][92],
                              "unconverged": [u for u in unc if u][:64]}), flush=True)
        except somf_pkg.SomfError as e:
            import numpy as np
            # k_bcd_big at its round cap: the first unconverged position's state
            st = np.array(cyc["raw"][72:80], dtype=np.int64).view(np.float64).tolist()
            print(json.dumps({"cfg": args.cfg, "r": args.r, "t": t + 1, "ok": False, "err": str(e),
                              "bcd": m.bcd_variant, "unconverged": unc[:64], "prefix_regressions": cyc["raw"][92],
                              "cap_state": dict(zip(("p+1000nmode+1e5mode", "lam", "nlam", "cnt", "min_above",
                                                     "max_below", "rho", "S1"), st)),
                              "first_unconverged": cyc["first_unconverged_per_round"],
                              "lam_first": np.array(cyc["raw"][96:160], dtype=np.int64).view(np.float64).tolist(),
                              "nlam_first": np.array(cyc["raw"][160:224], dtype=np.int64).view(np.float64).tolist()}),
                  flush=True)
            break


if __name__ == "__main__":
    main()
