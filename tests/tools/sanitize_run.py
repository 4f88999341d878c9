"""Developer harness for compute-sanitizer (racecheck / synccheck / memcheck):
a few SOMF steps of small shapes through every BCD / code / B-bar kernel
family, so that the hand-rolled grid barriers, PDL launches, cooperative
kernels and fixed-point atomics run under the tool.

    compute-sanitizer --tool racecheck python tests/tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1701_05363_b200 as somf  # noqa: E402

CASES = [
    # p, k, eta, kwargs
    (256, 10, 10, dict(lam=0.1, nu=1.0, mu=0.0, r=4.0, u=0.95)),                                    # cfgA
    (3000, 24, 40, dict(lam=1e-3, nu=1.0, mu=0.0, r=12.0)),                                         # ridge / l1
    (1536, 40, 32, dict(lam=0.1, nu=0.0, mu=1.0, r=4.0)),                                           # lasso / l2
    (2048, 24, 48, dict(lam=0.05, nu=1.0, pos_code=True, mu=1.0, pos_dict=True, r=8.0)),           # nmf
    (1520, 160, 33, dict(lam=0.05, nu=0.0, mu=0.5, r=3.0)),                                         # k > 128
]


def main():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    steps = int(os.environ.get("SAN_STEPS", "3"))
    for p, k, eta, kw in CASES:
        for bcd in ("auto", "onchip", "global", "big"):
            for b_mode in ("masked", "full", "unbiased"):
                X = torch.tensor(np.abs(rng.standard_normal((p, k + steps * eta))), dtype=torch.float32,
                                 device=dev)
                try:
                    m = somf.Somf(p, k, eta, seed=1, bcd_kernel=bcd, b_mode=b_mode, **kw)
                    m.set_components(X[:, :k].contiguous())
                    for t in range(steps):
                        m.partial_fit(X[:, k + t * eta:k + (t + 1) * eta].contiguous())
                    m.objective(X[:, :eta].contiguous())
                    st = m.get_state()
                except somf.SomfError as e:
                    print(f"skip p={p} k={k} {bcd} {b_mode}: {e}")
                    continue
                assert np.isfinite(st["D"]).all()
                torch.cuda.synchronize()
                print(f"ok p={p} k={k} eta={eta} bcd={m.bcd_variant} b_mode={b_mode}", flush=True)


if __name__ == "__main__":
    main()
