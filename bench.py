#!/usr/bin/env python
"""SOMF step throughput on B200 -- the BASELINE.json metric.

metric: streamed columns/sec of the SOMF step (one iteration of Alg. 3 + Alg. 4
of arXiv 1701.05363 on an eta-column mini-batch), with the roofline fraction
of the dominant kernel.  Workload (BASELINE.json configs[2], the config the
north star's >= 60 % target is quoted on): fMRI-shaped, p = 212445 voxels,
k = 70, eta = 200, r = 12, ridge lambda = 1e-3, l1-ball atoms (DESIGN.md §3
states the synthetic recipe; no HCP data is used).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl somf|reference]

A "step" is one somf_partial_fit on a batch resident in HBM; L2 is flushed
(256 MiB write) before every timed step, outside the step's CUDA events.
`e2e` times the same call with the batch in pinned HOST memory (the library
gathers the q selected rows over the host link) plus the device->host read of
the step's codes.  `--impl reference` times the float64 CPU oracle on the same
workload (bounded sample).  N > 1 (torchrun): one rank per
GPU, each owning rows [p i / N, p (i+1) / N) of D, Bbar and every batch; the
library's exchange points ([beta | G], radius sums, per-round threshold sums)
go through an NCCL allreduce; value = the job's columns/s.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(name="cfgC-fmri", p=212445, k=70, eta=200, lam=1e-3, nu=1.0, mu=0.0,
                pos_code=False, pos_dict=False, r=12.0, u=0.917)
METRIC = "streamed columns/sec (SOMF step)"
UNIT = "columns/s"
L2_FLUSH_BYTES = 256 << 20


# ----------------------------------------------------------------------------
# inputs (synthetic, seeded) -- shared with tests/test_gpu_parity.py
# ----------------------------------------------------------------------------
def fmri_inputs_cpu(n_cols: int, seed: int = 0, k: int = WORKLOAD["k"]):
    """(X p x n_cols, D0 p x k) float32 numpy: the first k stream columns
    initialise D (reading R15), the rest are batches."""
    import synth
    S = synth.fmri_stream(n_cols + k, seed=seed)
    return np.ascontiguousarray(S[:, k:]), np.ascontiguousarray(S[:, :k])


class FmriStreamGPU:
    """cfgC stand-in generated on the GPU (torch, harness only): batch b is
    D* a_b + noise, a_b the columns [k + b eta, k + (b+1) eta) of the AR(1)
    codes; D0 = the first k stream columns (reading R15)."""

    def __init__(self, n_batches: int, eta: int, k: int, seed: int, device):
        import torch
        import synth
        coords = synth.fmri_voxel_grid()
        self.p = coords.shape[0]
        self.eta, self.k, self.device = eta, k, device
        self.Dstar = torch.tensor(synth.fmri_dictionary(coords, 70, seed=seed), dtype=torch.float32,
                                  device=device)
        n = n_batches * eta + k
        self.A = torch.tensor(synth.fmri_codes(70, 1, T=max(1200, n), seed=seed + 1)[:, :n],
                              dtype=torch.float32, device=device)
        self.g = torch.Generator(device=device)
        self.g.manual_seed(seed + 2)
        self.sigma = float(np.sqrt(70 / self.p / 0.5))
        self.n_batches = n_batches

    def _cols(self, c0, c1):
        import torch
        X = self.Dstar @ self.A[:, c0:c1]
        X += self.sigma * torch.randn(X.shape, generator=self.g, device=self.device)
        return X.contiguous()

    def d0(self):
        return self._cols(0, self.k)

    def batch(self, b):
        b %= self.n_batches
        return self._cols(self.k + b * self.eta, self.k + (b + 1) * self.eta)


class HyperspectralStreamGPU:
    """cfgB stand-in on the GPU (harness only): 16 x 16 pixels x
    224 bands (p = 57,344, row = pixel * 224 + band); 256 |GP(RBF, l=20)|
    spectra (drawn once as in synth.hyperspectral_patches); every column mixes
    them with Dirichlet(0.5) abundances per pixel, 1 % Gaussian noise relative
    to the column rms, then is centred and l2-normalised."""

    def __init__(self, eta: int, seed: int, device, size: int = 16, bands: int = 224, n_end: int = 256):
        import torch
        rng = np.random.default_rng(seed)
        bb = np.arange(bands, dtype=np.float64)
        K = np.exp(-0.5 * ((bb[:, None] - bb[None, :]) / 20.0) ** 2)
        L = np.linalg.cholesky(K + 1e-8 * np.eye(bands))
        spectra = np.abs(L @ rng.standard_normal((bands, n_end))).T
        self.spectra = torch.tensor(spectra, dtype=torch.float32, device=device)      # n_end x bands
        self.npix, self.bands, self.eta, self.device = size * size, bands, eta, device
        self.p = self.npix * bands
        self.dir = torch.distributions.Dirichlet(torch.full((n_end,), 0.5, device=device))
        self.g = torch.Generator(device=device)
        self.g.manual_seed(seed + 1)
        torch.manual_seed(seed + 2)

    def batch(self, m: int | None = None):
        import torch
        m = m or self.eta
        ab = self.dir.sample((m, self.npix))                         # m x npix x n_end
        X = (ab @ self.spectra).reshape(m, self.p)                   # column s = row s here
        rms = X.pow(2).mean(dim=1, keepdim=True).sqrt()
        X = X + 0.01 * rms * torch.randn(X.shape, generator=self.g, device=self.device)
        X = X - X.mean(dim=1, keepdim=True)
        X = X / X.norm(dim=1, keepdim=True)
        return X.t().contiguous()                                    # p x m


class NmfStreamGPU:
    """cfgD stand-in on the GPU: X = W* H* + |N(0, 0.01)|, W* 16,384 x 128 |N(0,1)|
    at 30 % density (fixed), H* ~ Exp(1) per column."""

    def __init__(self, eta: int, seed: int, device, p: int = 16384, k_true: int = 128):
        import torch
        self.g = torch.Generator(device=device)
        self.g.manual_seed(seed)
        W = torch.randn((p, k_true), generator=self.g, device=device).abs()
        W *= (torch.rand((p, k_true), generator=self.g, device=device) < 0.3).float()
        self.W, self.p, self.k_true, self.eta, self.device = W, p, k_true, eta, device

    def batch(self, m: int | None = None):
        import torch
        m = m or self.eta
        H = torch.empty((self.k_true, m), device=self.device).exponential_(1.0, generator=self.g)
        N = (0.1 * torch.randn((self.p, m), generator=self.g, device=self.device)).abs()
        return (self.W @ H + N).contiguous()


class FmriEStreamGPU:
    """cfgE stand-in on the GPU (harness only): the cfgC recipe
    on a 126 x 160 x 100 grid masked to 2,000,000 voxels (synth.fmri_voxel_grid)
    with 256 truncated Gaussian blobs (centres uniform over the voxels, sigma ~
    U[2, 6], cut at 3 sigma, unit l2; built on the GPU: a dense float64 D* on
    the host would be 4 GB), AR(1) rho = 0.8 codes (synth.fmri_codes), SNR 0.5."""

    def __init__(self, eta: int, seed: int, device, k_true: int = 256, p: int = 2_000_000):
        import torch
        import synth
        coords = torch.tensor(synth.fmri_voxel_grid((126, 160, 100), p), dtype=torch.float32, device=device)
        self.p = coords.shape[0]
        rng = np.random.default_rng(seed)
        D = torch.zeros((self.p, k_true), dtype=torch.float32, device=device)
        for j in range(k_true):
            c = coords[int(rng.integers(self.p))]
            sg = float(rng.uniform(2.0, 6.0))
            d2 = ((coords - c) ** 2).sum(dim=1)
            v = torch.exp(-d2 / (2.0 * sg * sg))
            v[d2 > (3.0 * sg) ** 2] = 0.0
            D[:, j] = v / v.norm()
        self.Dstar = D
        self.A = torch.tensor(synth.fmri_codes(k_true, 1, T=4096, seed=seed + 1), dtype=torch.float32,
                              device=device)
        self.g = torch.Generator(device=device)
        self.g.manual_seed(seed + 2)
        self.sigma = float(np.sqrt(k_true / self.p / 0.5))
        self.eta, self.device, self.c0 = eta, device, 0

    def batch(self, m: int | None = None):
        import torch
        m = m or self.eta
        c0 = self.c0 % (self.A.shape[1] - m)
        self.c0 += m
        X = self.Dstar @ self.A[:, c0:c0 + m]
        X += self.sigma * torch.randn(X.shape, generator=self.g, device=self.device)
        return X.contiguous()


def fmri_inputs_gpu(n_batches: int, eta: int, k: int, seed: int, device):
    """(list of p x eta float32 CUDA batches, D0 p x k) of FmriStreamGPU."""
    s = FmriStreamGPU(n_batches, eta, k, seed, device)
    D0 = s.d0()
    return [s.batch(b) for b in range(n_batches)], D0


# ----------------------------------------------------------------------------
# roofline bookkeeping: algorithmic bytes / flops per launch
# ----------------------------------------------------------------------------
def phase_cost(phase: str, q: float, p: int, k: int, eta: int):
    """(bytes, flops, bound) of one launch of the phase's dominant kernel."""
    if phase == "contract":   # read D_M, X_M, idx; (beta | G) outputs are tiny
        return 4 * q * (k + eta + 1), 2 * q * k * (eta + k), "hbm"
    if phase == "bbar":       # read X_M, idx; read + write Bbar_M
        return 4 * q * (eta + 2 * k + 1), 2 * q * k * eta, "hbm"
    if phase == "bcd":        # read + write D_M, read Bbar_M, idx
        return 4 * q * (3 * k + 1), 2 * q * k * k, "hbm"
    if phase == "codes":
        return 8 * (k * k + 2 * k * eta), k ** 3 / 3 + 2 * k * k * eta, "alu"
    if phase == "cbar":
        return 8 * (2 * k * k + k * eta), 2 * k * k * eta, "alu"
    if phase == "mask":
        return 4 * q, 0.0, "hbm"
    if phase == "stage":
        return 8 * q * eta, 0.0, "hbm"
    raise KeyError(phase)


def step_bytes(q: float, k: int, eta: int):
    """4q(4k + eta) + 8q bytes per iteration (masked modes)."""
    return 4 * q * (4 * k + eta) + 8 * q


def step_roofline_us(q: float, k: int, eta: int, peaks: dict) -> float:
    """SURVEY §8(d) step roofline: the slower of the algorithmic bytes over HBM
    and the contractions on the tensor pipe (3xTF32: 3 x (4 q k eta + q k^2)
    at the TF32 rate = measured bf16 / 2) plus the BCD recurrence on FFMA
    (2 q k^2 + 10 q k at the fp32 CUDA-core peak)."""
    t_hbm = step_bytes(q, k, eta) / (peaks["hbm"] * 1e9)
    t_tc = 3.0 * (4 * q * k * eta + q * k * k) / (peaks["bf16"] / 2.0 * 1e12)
    t_fma = (2 * q * k * k + 10 * q * k) / (alu_peak_tflops(peaks["sm_max_mhz"], fp64=False) * 1e12)
    return 1e6 * max(t_hbm, t_tc + t_fma)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        mp = json.load(open(path))
        return dict(hbm=mp["hbm_gbs"], bf16=mp["bf16_tflops"], src="measured",
                    sm_max_mhz=mp.get("sm_max_mhz", 1965.0))
    return dict(hbm=6650.0, bf16=1590.0, src="fallback", sm_max_mhz=1965.0)


def alu_peak_tflops(sm_mhz: float, fp64: bool = True):
    """CUDA-core FMA peak: 148 SMs x 128 FP32 lanes (64 FP64 lanes) x 2 x clock."""
    lanes = 64 if fp64 else 128
    return 148 * lanes * 2 * sm_mhz * 1e6 / 1e12


# ----------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ----------------------------------------------------------------------------
class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) polled every ~1 ms from a thread, so even a few-ms timed
    region gets samples; falls back to `nvidia-smi -lms 100`."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, cuda_index: int):
        self.cuda_index = cuda_index
        self.samples, self.maxc, self.reasons = [], None, set()
        self.stop_ev = threading.Event()
        self.th = None
        self.proc = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.cuda_index)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml.nvmlDeviceGetHandleByIndex(self.cuda_index)

    def _poll(self, h):
        import pynvml
        get_r = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_ev.is_set():
            try:
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                bits = get_r(h)
                for m, nm in self.REASONS.items():
                    if bits & m:
                        self.reasons.add(nm)
            except Exception:
                pass
            time.sleep(0.001)

    def start(self):
        try:
            import pynvml
            h = self._handle()
            self.maxc = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.th = threading.Thread(target=self._poll, args=(h,), daemon=True)
            self.th.start()
            time.sleep(0.003)            # at least one sample before the timed region
        except Exception:
            self.th = None
            try:
                q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                     "clocks_event_reasons.sw_power_cap")
                self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.cuda_index}", f"--query-gpu={q}",
                                              "--format=csv,noheader,nounits", "-lms", "100"],
                                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            except (OSError, FileNotFoundError):
                self.proc = None

    def stop(self):
        if self.th is not None:
            time.sleep(0.002)
            self.stop_ev.set()
            self.th.join(timeout=2)
            if not self.samples:
                return None
            return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.maxc,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml 1 ms"}
        if self.proc is None:
            return None
        self.proc.terminate()
        out = self.proc.communicate(timeout=5)[0]
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in out.splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi 100 ms"}


# ----------------------------------------------------------------------------
# CPU oracle leg
# ----------------------------------------------------------------------------
def oracle_throughput(batches_cpu, D0, budget_s: float, max_steps: int, warm: int = 1):
    """Time the float64 oracle (as it stands) on host cores: returns
    (columns/s, steps timed, seconds)."""
    from oracle.somf import SomfOracle, OracleConfig
    w = WORKLOAD
    ora = SomfOracle(OracleConfig(p=w["p"], k=w["k"], eta=w["eta"], lam=w["lam"], nu=w["nu"],
                                  mu=w["mu"], r=w["r"], u=w["u"], seed=0))
    ora.set_components(D0)
    i = 0
    for _ in range(warm):
        ora.partial_fit(batches_cpu[i % len(batches_cpu)])
        i += 1
    t0 = time.perf_counter()
    n = 0
    while n < max_steps and (time.perf_counter() - t0) < budget_s:
        ora.partial_fit(batches_cpu[i % len(batches_cpu)])
        i += 1
        n += 1
    dt = time.perf_counter() - t0
    return w["eta"] * n / dt, n, dt


def host_cores():
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count()
    threads = None
    try:
        from threadpoolctl import threadpool_info
        threads = max((i.get("num_threads", 0) for i in threadpool_info()), default=None)
    except Exception:
        pass
    return cores, threads


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = WORKLOAD
    X, D0 = fmri_inputs_cpu(4 * w["eta"], seed=0)
    batches = [X[:, i * w["eta"]:(i + 1) * w["eta"]] for i in range(4)]
    val, n, dt = oracle_throughput(batches, D0, budget_s=max(30.0, 8.0 * args.steps),
                                   max_steps=args.steps, warm=args.warmup)
    cores, threads = host_cores()
    sample = f"{n} oracle steps of {w['name']} r={w['r']} after {args.warmup} warm-up steps (pool of 4 batches)"
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": n, "warmup": args.warmup, "ms_per_step": 1e3 * dt / max(n, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (fMRI-shaped, DESIGN.md §3)",
            "config": {"workload": w["name"], "p": w["p"], "k": w["k"], "eta": w["eta"], "r": w["r"]},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "blas_threads": threads,
                             "kind": "oracle", "sample": sample},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# GPU leg
# ----------------------------------------------------------------------------
def time_steps(model, batches, start, steps, flush, stream):
    """Per-step CUDA-event durations (ms) with an L2 flush before each step."""
    import torch
    evs = []
    for i in range(steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        model.partial_fit(batches[(start + i) % len(batches)])
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in evs]


def run_somf(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # ranks beyond the visible GPUs share them (only with --dist-backend gloo:
    # a host-side collective, no kernel waits on another rank)
    dev = torch.device("cuda", local % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    if world > 1:
        if args.dist_backend == "nccl" and world > torch.cuda.device_count():
            raise SystemExit(f"--gpus {world} with NCCL needs {world} visible GPUs "
                             f"({torch.cuda.device_count()} found); use --dist-backend gloo to share one")
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    import paper_1701_05363_b200 as somf_pkg
    somf_pkg.lib()
    w = WORKLOAD
    p, k, eta, r = w["p"], w["k"], w["eta"], args.r
    stream = torch.cuda.current_stream(dev)
    nb = min(args.warmup + args.steps, 24)
    # every rank draws the same stream and keeps its row range [lo, hi) (row
    # sharding): the job streams eta columns per step over all ranks
    stream_gen = FmriStreamGPU(args.burn_in + nb, eta, k, seed=0, device=dev)
    lo, hi = p * rank // world, p * (rank + 1) // world
    D0 = stream_gen.d0()[lo:hi]
    # the timed pool: the batches that follow the burn-in in the stream
    batches = [stream_gen.batch(args.burn_in + b)[lo:hi] for b in range(nb)]
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)

    def make(rr, burn_in, b_mode="masked"):
        m = somf_pkg.Somf(p, k, eta, lam=w["lam"], nu=w["nu"], mu=w["mu"], pos_code=w["pos_code"],
                          row_lo=lo, row_hi=hi, b_mode=b_mode, bcd_copies=args.bcd_copies,
                          pos_dict=w["pos_dict"], r=rr, u=w["u"], seed=0, device=dev.index, stream=stream)
        if world > 1:
            m.set_reducer(somf_pkg.dist_reducer())      # NCCL allreduce at every exchange point
        m.set_components(D0)
        # burn-in: the learner reaches its steady state (t > burn_in) on fresh
        # stream batches before anything is timed (steady state)
        for b in range(burn_in):
            m.partial_fit(stream_gen.batch(b)[lo:hi])
        return m

    model = make(r, args.burn_in)
    for i in range(args.warmup):
        model.partial_fit(batches[i % nb])
    torch.cuda.synchronize()
    model.profile_read()
    model.profile_enable(False)
    clocks = Clocks(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t_wall = time.perf_counter()
    ms = time_steps(model, batches, args.warmup, args.steps, flush, stream)
    t_wall = time.perf_counter() - t_wall
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    launch_counts = model.profile_read()     # launches of the timed (unprofiled) steps
    info = model.last_step_info()
    # per-kernel durations: the same number of steps again with CUDA events
    # around every phase on the launching stream (kept out of the timed value)
    model.profile_enable(True)
    time_steps(model, batches, args.warmup + args.steps, args.steps, flush, stream)
    prof = model.profile_read()
    bcd_cyc = model.bcd_phase_cycles()
    model.profile_enable(False)
    prof["launches"] = launch_counts["launches"]
    # host time of one somf_partial_fit call (enqueue only: argument checks,
    # by-value parameters, launches), the GPU working behind it
    torch.cuda.synchronize()
    host_us = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        model.partial_fit(batches[(2 * args.steps + args.warmup + i) % nb])
        host_us.append((time.perf_counter() - t0) * 1e6)
    torch.cuda.synchronize()
    step_ms = sum(ms) / len(ms)
    if world > 1:
        tt = torch.tensor([step_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        step_ms = float(tt.item())
    value = eta / (step_ms * 1e-3)      # the job's columns per second (all ranks share each column)

    # --- roofline of the dominant kernel ------------------------------------
    q = p / r
    peaks = measured_peaks()
    steps_prof = max(prof["steps"], 1)
    phase_ms = {ph: prof["ms"][ph] / steps_prof for ph in prof["ms"]}
    dom = max(phase_ms, key=lambda ph: phase_ms[ph])
    by, fl, bound = phase_cost(dom, q, p, k, eta)
    dom_ms = phase_ms[dom]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(dom)
    if bound == "hbm":
        achieved = by / (dom_ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm"], "unit": "GB/s",
                "frac": achieved / peaks["hbm"], "traffic": traffic, "kernel_phase": dom,
                "peak_source": peaks["src"]}
    else:
        achieved = fl / (dom_ms * 1e-3) / 1e12
        pk = alu_peak_tflops(peaks["sm_max_mhz"], fp64=True)
        roof = {"bound": "alu", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
                "frac": achieved / pk, "traffic": traffic, "kernel_phase": dom,
                "peak_source": "guide: 148 SM x 64 FP64 lanes x 2 x sm_max_mhz"}
    roof["phase_ms_per_step"] = phase_ms
    # every phase against its own bound: algorithmic bytes over
    # HBM, the contractions' algorithmic flops over the tensor-core peak of the
    # dtype they run in (3xTF32 / bf16x3 issue 3 products per flop counted once),
    # the BCD also against the CUDA-core fp32 FMA peak (its recurrence pipe)
    tf32_peak = peaks["bf16"] / 2.0          # guide: dense TF32 = 1/2 dense BF16
    per = {}
    for ph, pms in phase_ms.items():
        if pms <= 0 or ph in ("stage", "mask", "cbar"):
            continue
        pb, pf, _ = phase_cost(ph, q, p, k, eta)
        ent = {"ms": pms, "hbm_gbs": pb / (pms * 1e-3) / 1e9, "hbm_frac": pb / (pms * 1e-3) / 1e9 / peaks["hbm"]}
        if ph == "contract":
            ent.update(tensor_tflops=pf / (pms * 1e-3) / 1e12, tensor_peak=tf32_peak, tensor_dtype="tf32 (3xTF32)",
                       tensor_frac=pf / (pms * 1e-3) / 1e12 / tf32_peak)
        if ph == "bbar":
            ent.update(tensor_tflops=pf / (pms * 1e-3) / 1e12, tensor_peak=peaks["bf16"], tensor_dtype="bf16 (bf16x3)",
                       tensor_frac=pf / (pms * 1e-3) / 1e12 / peaks["bf16"])
        if ph == "bcd":
            fp32 = alu_peak_tflops(peaks["sm_max_mhz"], fp64=False)
            ent.update(fma_tflops=pf / (pms * 1e-3) / 1e12, fma_peak=fp32, fma_frac=pf / (pms * 1e-3) / 1e12 / fp32)
        per[ph] = ent
    roof["phases"] = per
    roof["bcd_grid_reductions_per_step"] = info["bcd_reductions"]
    if bcd_cyc["launches"]:
        mhz = (clk or {}).get("sm_mhz") or peaks["sm_max_mhz"]
        roof["bcd_phase_us_per_step"] = {ph: v / bcd_cyc["launches"] / mhz for ph, v in bcd_cyc.items()
                                         if isinstance(v, int) and ph not in ("launches", "unconverged_per_round", "frozen_prefix_per_round", "ridge",
                                                       "setup_split", "update_split", "contract", "bbar")}
        roof["bcd_update_us_per_step"] = {ph: v / bcd_cyc["launches"] / mhz for ph, v in bcd_cyc["update_split"].items()}
        roof["ridge_phase_us_per_step"] = {ph: v / bcd_cyc["launches"] / mhz for ph, v in bcd_cyc["ridge"].items()}
        for ph in ("contract", "bbar"):
            n = bcd_cyc[ph].pop("launches")
            if n:
                roof[ph + "_phase_us_per_step"] = {x: v / n / mhz for x, v in bcd_cyc[ph].items()}
        roof["bcd_setup_us_per_step"] = {ph: v / bcd_cyc["launches"] / mhz for ph, v in bcd_cyc["setup_split"].items()}
        unc = [u / bcd_cyc["launches"] for u in bcd_cyc["unconverged_per_round"]]
        while unc and unc[-1] == 0:
            unc.pop()
        roof["bcd_unconverged_atoms_per_round"] = [round(u, 2) for u in unc]
        roof["bcd_frozen_prefix_per_round"] = [round(f / bcd_cyc["launches"], 2)
                                               for f in bcd_cyc["frozen_prefix_per_round"][:len(unc)]]
    sb = step_bytes(q, k, eta)
    roof_us = step_roofline_us(q, k, eta, peaks)
    step_roof = {"bytes_per_step": sb, "achieved_gbs": sb / (step_ms * 1e-3) / 1e9,
                 "frac_of_hbm": sb / (step_ms * 1e-3) / 1e9 / peaks["hbm"],
                 "roofline_us": roof_us, "frac": roof_us / (step_ms * 1e3)}

    # --- end-to-end through the C ABI with host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        n_e2e = min(args.steps, 10)
        host = [b.cpu().pin_memory() for b in batches[:2]]
        codes = torch.empty((k, eta), dtype=torch.float32).pin_memory()
        m2 = make(r, args.burn_in)
        for i in range(2):
            m2.partial_fit(host[i % 2])
        torch.cuda.synchronize()
        qs, times = [], []
        for i in range(n_e2e):
            flush.zero_()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            m2.partial_fit(host[i % 2])
            m2.get_codes(codes)
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
            qs.append(m2.last_step_info()["q"])
        e_ms = sum(times) / len(times)
        e2e = {"value": eta / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(4 * eta * sum(qs) / len(qs)), "d2h_bytes_per_step": 4 * k * eta,
               "ms_per_step": e_ms, "path": "somf_partial_fit(pinned host X) + somf_get_codes(host)"}
        del m2

    # --- r sweep (BASELINE metric lists r = 1/4/12/24) ---------------------------
    sweep = {}
    if not args.no_sweep and world == 1:
        for rr in (1.0, 4.0, 12.0, 24.0):
            m3 = make(rr, args.burn_in if rr > 1.0 else min(args.burn_in, 10))
            for i in range(3):
                m3.partial_fit(batches[i % nb])
            torch.cuda.synchronize()
            t3 = time_steps(m3, batches, 3, 5, flush, stream)
            sm = sum(t3) / len(t3)
            sweep[f"r={int(rr)}"] = {"columns_per_s": eta / (sm * 1e-3), "ms_per_step": sm,
                                     "roofline_us": step_roofline_us(p / rr, k, eta, measured_peaks()),
                                     "roofline_frac": step_roofline_us(p / rr, k, eta, measured_peaks()) / (sm * 1e3),
                                     "bcd_kernel": m3.bcd_variant,
                                     "bcd_grid_reductions": m3.last_step_info()["bcd_reductions"]}
            del m3
        # mode F (Alg. 3 as printed): the rows outside M_t also update
        # their Bbar, on a side stream beside the BCD
        m3 = make(r, args.burn_in, b_mode="full")
        for i in range(3):
            m3.partial_fit(batches[i % nb])
        torch.cuda.synchronize()
        t3 = time_steps(m3, batches, 3, 5, flush, stream)
        sm = sum(t3) / len(t3)
        sweep[f"r={int(r)} b_mode=full"] = {"columns_per_s": eta / (sm * 1e-3), "ms_per_step": sm,
                                             "bcd_kernel": m3.bcd_variant,
                                             "bcd_grid_reductions": m3.last_step_info()["bcd_reductions"]}
        del m3

    # --- the other BASELINE workloads (single GPU, secondary lines) -----------------
    # cfgB hyperspectral (k = 256, lasso codes, l2-ball atoms) at r = 1/4/12 and
    # cfgD NMF (k = 128, nonneg ridge CD codes, nonneg l2-ball atoms) at r = 8:
    # 10 burn-in steps from the first k stream columns, then 5 timed steps
    workloads = {}
    if not args.no_sweep and world == 1:
        specs = [("cfgB-hyperspectral", HyperspectralStreamGPU, 256, 256,
                  dict(lam=0.1, nu=0.0, mu=1.0, pos_code=False, pos_dict=False), (1.0, 4.0, 12.0)),
                 ("cfgD-nmf", NmfStreamGPU, 128, 512,
                  dict(lam=0.05, nu=1.0, mu=1.0, pos_code=True, pos_dict=True), (8.0,)),
                 ("cfgE-fmri2M", FmriEStreamGPU, 256, 512,
                  dict(lam=0.05, nu=0.0, mu=0.5, pos_code=False, pos_dict=False), (24.0, 12.0, 4.0))]
        for name, gen_cls, kk, ee, kw, rs in specs:
            gen = gen_cls(ee, seed=0, device=dev)
            pool = [gen.batch() for _ in range(8)]
            d0 = gen.batch(kk)
            res = {}
            for rr in rs:
                try:
                    m4 = somf_pkg.Somf(gen.p, kk, ee, r=rr, u=w["u"], seed=0, device=dev.index, stream=stream, **kw)
                    m4.set_components(d0)
                    for i in range(10):
                        m4.partial_fit(pool[i % len(pool)])
                    torch.cuda.synchronize()
                    t4 = time_steps(m4, pool, 10, 5, flush, stream)
                    sm4 = sum(t4) / len(t4)
                    info4 = m4.last_step_info()
                    m4.profile_read()
                    m4.profile_enable(True)
                    time_steps(m4, pool, 15, 3, flush, stream)
                    pr4 = m4.profile_read()
                    m4.profile_enable(False)
                    roof4 = step_roofline_us(gen.p / rr, kk, ee, measured_peaks())
                    res[f"r={int(rr)}"] = {"columns_per_s": ee / (sm4 * 1e-3), "ms_per_step": sm4,
                                           "roofline_us": roof4, "roofline_frac": roof4 / (sm4 * 1e3),
                                           "bcd_kernel": m4.bcd_variant,
                                           "bcd_grid_reductions": info4["bcd_reductions"], "q": info4["q"],
                                           "phase_ms_per_step": {ph: v / max(pr4["steps"], 1)
                                                                 for ph, v in pr4["ms"].items() if v > 0}}
                    del m4
                except somf_pkg.SomfError as e:
                    # a secondary line must not take the headline down: record the failure
                    res[f"r={int(rr)}"] = {"error": str(e)}
                    print(f"bench: workload {name} r={rr} failed: {e}", file=sys.stderr, flush=True)
            workloads[name] = {"p": gen.p, "k": kk, "eta": ee, **{k_: v for k_, v in kw.items()}, "results": res}

    # --- CPU oracle baseline (rank 0, N = 1) ----------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        hb = [b.cpu().numpy() for b in batches[:3]]
        val, n, dt = oracle_throughput(hb, D0.cpu().numpy(), budget_s=args.cpu_budget, max_steps=50)
        cores, threads = host_cores()
        cpu = {"value": val, "unit": UNIT, "cores": cores, "blas_threads": threads, "kind": "oracle",
               "sample": f"{n} float64 oracle steps ({dt:.1f} s) of the same workload after 1 warm-up step"}

    launches = int(sum(prof["launches"].values()))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "ms_per_step_median": statistics.median(ms),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (fMRI-shaped stand-in, DESIGN.md §3)",
            "config": {"workload": w["name"], "p": p, "k": k, "eta": eta, "r": r, "lambda": w["lam"],
                       "code": "ridge", "dict": "l1-ball", "b_mode": "masked",
                       "bcd_kernel": model.bcd_variant,
                       "l2": "flushed (256 MiB write) before every timed step",
                       "burn_in_iterations": args.burn_in,
                       "parallelism": "single" if world == 1 else f"row-sharded x{world} ({args.dist_backend} allreduce)"},
            "roofline": roof, "step_roofline": step_roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "gpu_launches_per_step": launches / steps_prof,
            "host_us_per_call": statistics.median(host_us),
            "clocks": clk, "sweep": sweep, "workloads": workloads, "wall_s_timed": t_wall}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------
# time-to-1 % sweeps (Table III; validation
# protocol P:1322-1326): OMF (r = 1) vs SOMF r in {4, 12, 24}
# ----------------------------------------------------------------------------
def convergence_curve(model, X_all, ids_of, iters, eval_every, Xte, stream, use_ids=True):
    """Runs `iters` steps of `model` on batches X_all[:, ids_of(t)] and returns
    [(cumulative step time in s, iteration, test objective)] at every
    `eval_every` steps (and at 0).  Only the partial_fit calls are timed (CUDA
    events on the launching stream); gathers of the batch and the objective
    evaluations are outside the timed region."""
    import torch
    curve = [(0.0, 0, model.objective(Xte))]
    t_acc = 0.0
    for t in range(iters):
        ids = ids_of(t)
        batch = X_all[:, ids].contiguous()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        if use_ids:
            model.partial_fit_ids(batch, ids)
        else:
            model.partial_fit(batch)
        b.record(stream)
        b.synchronize()
        t_acc += a.elapsed_time(b) * 1e-3
        if (t + 1) % eval_every == 0 or t + 1 == iters:
            curve.append((t_acc, t + 1, model.objective(Xte)))
    return curve


def time_to_within(curve, f_star, tol=0.01):
    """First (time, iteration) with test objective <= (1 + tol) f_star, else None."""
    for tm, it, f in curve:
        if f <= (1.0 + tol) * f_star:
            return tm, it
    return None


def run_sweeps(args):
    """cfgC stand-in (fMRI-shaped, p = 212,445, k = 70, eta = 200, ridge
    lambda = 1e-3, l1-ball atoms): a finite set of n columns cycled randomly
    (per-epoch keyed permutations, reading R16, the same order for every r,
    P:1354-1357), estimator (c) (the paper's choice on fMRI),
    held-out objective on 1000 other columns against step time; time to reach
    1 % of the best objective any run reached (Table III's criterion)."""
    import torch
    import paper_1701_05363_b200 as somf_pkg
    somf_pkg.lib()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    w = WORKLOAD
    p, k, eta = w["p"], w["k"], w["eta"]
    n, n_te = args.sweep_n, 1000
    gen = FmriStreamGPU(n_batches=(n + n_te) // eta + 1, eta=eta, k=k, seed=5, device=dev)
    X_all = gen._cols(k, k + n)                        # p x n (the data set)
    Xte = gen._cols(k + n, k + n + n_te)               # held-out columns
    D0 = gen._cols(0, k)
    stream = torch.cuda.current_stream(dev)

    def ids_of(t):
        return somf_pkg.column_ids(11, n, t * eta, eta)

    curves, step_ms = {}, {}
    for rr in args.sweep_r:
        m = somf_pkg.Somf(p, k, eta, lam=w["lam"], nu=w["nu"], mu=w["mu"], r=rr, u=w["u"], seed=0,
                          estimator=args.sweep_estimator, n_samples=n, device=0, stream=stream)
        m.set_components(D0)
        iters = args.sweep_iters
        cv = convergence_curve(m, X_all, ids_of, iters, args.sweep_eval, Xte, stream,
                               use_ids=args.sweep_estimator != "a")
        curves[f"r={int(rr)}"] = cv
        step_ms[f"r={int(rr)}"] = 1e3 * cv[-1][0] / iters
        del m
    f_star = min(f for cv in curves.values() for _, _, f in cv)
    out = {}
    for name, cv in curves.items():
        hit = time_to_within(cv, f_star, 0.01)
        out[name] = {"ms_per_step": step_ms[name], "final_objective": cv[-1][2],
                     "time_to_1pct_s": hit[0] if hit else None, "iters_to_1pct": hit[1] if hit else None,
                     "curve": [[round(tm, 6), it, f] for tm, it, f in cv]}
    base = out.get("r=1", {}).get("time_to_1pct_s")
    for name, o in out.items():
        o["speedup_vs_omf"] = (base / o["time_to_1pct_s"]) if (base and o["time_to_1pct_s"]) else None
    line = {"metric": "time to 1% of the best test objective (OMF r=1 vs SOMF)", "unit": "s (device time of the steps)",
            "workload": "cfgC-fmri", "p": p, "k": k, "eta": eta, "n_columns": n, "n_test": n_te,
            "estimator": args.sweep_estimator, "f_star": f_star, "iters": args.sweep_iters,
            "eval_every": args.sweep_eval, "data": "synthetic (fMRI-shaped stand-in, DESIGN.md §3)", "results": out}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="somf", choices=["somf", "reference"])
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collectives of the row-sharded step (gloo: CPU-staged, lets N ranks share one GPU)")
    ap.add_argument("--burn-in", type=int, default=60,
                    help="untimed SOMF iterations before warm-up (steady state, t > burn-in)")
    ap.add_argument("--r", type=float, default=WORKLOAD["r"])
    ap.add_argument("--bcd-copies", type=int, default=0,
                    help="copies of each per-atom BCD accumulator (performance knob; 0 = library default)")
    ap.add_argument("--sweeps", action="store_true",
                    help="time-to-1%% convergence sweeps (OMF r=1 vs SOMF r=4/12/24) instead of the step benchmark")
    ap.add_argument("--sweep-r", type=float, nargs="+", default=[1.0, 4.0, 12.0, 24.0])
    ap.add_argument("--sweep-n", type=int, default=12000)
    ap.add_argument("--sweep-iters", type=int, default=1200)
    ap.add_argument("--sweep-eval", type=int, default=20)
    ap.add_argument("--sweep-estimator", default="c", choices=["a", "b", "c"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: start the N ranks ourselves (the driver uses
        # torchrun; this keeps `python bench.py --gpus N` equivalent)
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    elif args.sweeps:
        run_sweeps(args)
    else:
        run_somf(args)


if __name__ == "__main__":
    main()
