"""Seeded synthetic inputs shaped like the paper's workloads.

This module is shared by the oracle-side tests and the CUDA path's tests and
bench.  It holds NONE of the method's arithmetic (no RNG streams of the
method, no quantisation, no trees): it only fabricates (X, y) arrays with a
numpy PCG64 generator.  Recipes are documented in DESIGN.md section 4.

paper_shaped(): 12 columns in the order of Table 6:
    threads per CTA, CTAs, total instr., special ops, logic ops, control ops,
    arithm. ops, sync ops, global mem vol., param mem vol., shared mem vol.,
    arithm. intensity.
  Targets per GPU of Table 3: time in microseconds spanning
  microseconds to seconds, power in watts within two orders of
  magnitude.  5 % of rows repeat the previous row's features with a
  different target (identical features for different samples).
scaled(): paper_shaped features + finer per-class sub-counts (the "possibly
  hundreds of features" of P:440-442) + 4 low-cardinality columns.
"""
from __future__ import annotations

import numpy as np

# Table 3: SMs, memory bandwidth GB/s, core clock MHz (GTX1650: top of range), TDP W
GPUS = {
    "K20": dict(sms=13, bw=208.0, clk=706.0, tdp=225.0, sigma=0.05),
    "TitanXp": dict(sms=30, bw=548.0, clk=1404.0, tdp=250.0, sigma=0.05),
    "P100": dict(sms=56, bw=732.0, clk=1189.0, tdp=300.0, sigma=0.05),
    "V100": dict(sms=80, bw=900.0, clk=1290.0, tdp=300.0, sigma=0.05),
    "GTX1650": dict(sms=14, bw=128.0, clk=2250.0, tdp=75.0, sigma=0.30),
}
GPU_NAMES = list(GPUS)
FEATURES = ["threads_per_cta", "ctas", "total_instr", "special_ops", "logic_ops", "control_ops",
            "arith_ops", "sync_ops", "global_mem_vol", "param_mem_vol", "shared_mem_vol",
            "arith_intensity"]
SEED = 20010710


def _features(rng, n):
    tpc = rng.choice([32, 64, 128, 192, 256, 512, 1024], size=n,
                     p=[.05, .15, .30, .05, .30, .10, .05]).astype(np.float64)
    ctas = np.round(10.0 ** rng.uniform(0.0, 5.5, size=n))
    ctas = np.maximum(ctas, 1.0)
    per_thread = 10.0 ** rng.uniform(1.0, 4.5, size=n)
    mix = rng.dirichlet([4.0, 2.0, 2.0, 0.5, 0.5, 3.0], size=n)  # arith, logic, control, special, sync, mem
    total = per_thread * tpc * ctas
    cls = np.round(mix * total[:, None])
    arith, logic, control, special, sync, mem = (cls[:, i] for i in range(6))
    gvol = np.round(mem * rng.choice([4.0, 8.0, 16.0], size=n) * rng.uniform(0.3, 1.0, size=n))
    pvol = np.round(10.0 ** rng.uniform(1.0, 3.0, size=n) * tpc * ctas)
    svol = np.round(mem * 4.0 * rng.uniform(0.0, 0.7, size=n))
    ai = arith / np.maximum(gvol, 1.0)
    tot = arith + logic + control + special + sync + mem
    X = np.stack([tpc, ctas, tot, special, logic, control, arith, sync, gvol, pvol, svol, ai], axis=1)
    return X, dict(arith=arith, special=special, mem=mem, gvol=gvol, tpc=tpc, ctas=ctas, sync=sync,
                   total=tot)


def _time_us(rng, parts, g):
    # compute term: instructions over (SMs * 64 lanes * clock); memory term: bytes / bandwidth
    lanes = g["sms"] * 64.0 * g["clk"] * 1e6
    comp = (parts["arith"] + 4.0 * parts["special"] + parts["total"] * 0.25) / lanes * 1e6
    memt = parts["gvol"] / (g["bw"] * 1e9) * 1e6
    sync = parts["sync"] / lanes * 1e6 * 8.0
    t = 2.0 + comp + memt + sync
    return t * np.exp(rng.normal(0.0, g["sigma"], size=t.shape[0]))


def _power_w(rng, parts, g):
    idle = 0.2 * g["tdp"]
    occ = np.minimum(1.0, parts["ctas"] * parts["tpc"] / (g["sms"] * 2048.0))
    frac = parts["arith"] / np.maximum(parts["total"], 1.0)
    memfrac = parts["gvol"] / np.maximum(parts["gvol"] + parts["arith"] * 4.0, 1.0)
    mixf = 0.35 + 0.45 * frac + 0.2 * memfrac
    pw = idle + (g["tdp"] - idle) * occ * mixf
    return pw * (1.0 + 0.01 * rng.normal(0.0, 1.0, size=pw.shape[0]))


def paper_shaped(n: int = 189, gpu: str = "K20", target: str = "time", seed: int = SEED):
    """(X [n,12] float64, y [n] float64 > 0).  time in us (LOG target), power in W."""
    gi = GPU_NAMES.index(gpu)
    rng = np.random.default_rng([seed, n, gi, 0 if target == "time" else 1])
    # features do not depend on the GPU (portable features)
    frng = np.random.default_rng([seed, n, 99, 0 if target == "time" else 1])
    X, parts = _features(frng, n)
    dup = frng.uniform(size=n) < 0.05
    dup[0] = False
    for i in np.nonzero(dup)[0]:
        X[i] = X[i - 1]
        for key in parts:
            parts[key][i] = parts[key][i - 1]
    g = GPUS[gpu]
    y = _time_us(rng, parts, g) if target == "time" else _power_w(rng, parts, g)
    return np.ascontiguousarray(X), np.ascontiguousarray(y)


def study(seed: int = SEED):
    """The full study inputs (config 'full study'): 5 GPUs x {time n=189, power n=168}."""
    out = []
    for gpu in GPU_NAMES:
        X, y = paper_shaped(189, gpu, "time", seed)
        out.append(dict(name=f"{gpu}/time", gpu=gpu, target="time", X=X, y=y))
        X, y = paper_shaped(168, gpu, "power", seed)
        out.append(dict(name=f"{gpu}/power", gpu=gpu, target="power", X=X, y=y))
    return out


def scaled(n: int, p: int = 64, seed: int = SEED):
    """Scaled synthetic set: paper features, sub-counts, 4 low-cardinality columns; K20 time target."""
    assert p >= 16
    rng = np.random.default_rng([seed, n, p, 7])
    X12, parts = _features(rng, n)
    nsub = p - 12 - 4
    cls = np.stack([X12[:, 6], X12[:, 4], X12[:, 5], X12[:, 3]], axis=1)
    sub = np.empty((n, nsub))
    for j in range(nsub):
        sub[:, j] = np.round(cls[:, j % 4] * rng.uniform(0.05, 0.5, size=n))
    low = rng.integers(0, 8, size=(n, 4)).astype(np.float64)
    X = np.concatenate([X12, sub, low], axis=1)
    y = _time_us(rng, parts, GPUS["K20"])
    return np.ascontiguousarray(X), np.ascontiguousarray(y)


def queries(n: int, p: int = 64, seed: int = SEED):
    """Held-out query rows for inference (seed + 1)."""
    return scaled(n, p, seed + 1)[0]


def tiny(n: int, p: int, seed: int, distinct: int | None = None, pos: bool = True):
    """Small random datasets for parity sweeps; `distinct` limits values per column (ties)."""
    rng = np.random.default_rng([seed, n, p, 11])
    if distinct:
        X = rng.integers(0, distinct, size=(n, p)).astype(np.float64)
    else:
        X = rng.normal(size=(n, p))
    y = rng.lognormal(0.0, 1.0, size=n) if pos else rng.normal(size=n)
    return np.ascontiguousarray(X), np.ascontiguousarray(y)


# ------------------------------------------------------ on-device generator --
# The C4 / C5 sets (10M / 100M rows x 64 features = 5.1 / 51 GB) are generated on the GPU with
# the same recipe as scaled() ("For C4/C5 an on-device generator
# may be used; the oracle then consumes the D2H copy of exactly those bytes").  torch's CUDA
# Philox generator, one generator per block of DEV_BLOCK rows seeded by (seed, block), so the
# rows of a block do not depend on n (a 10M-row set is the prefix of the 100M-row one) and the
# output is identical run to run.  Like the rest of this module it holds none of the method's
# arithmetic.
DEV_BLOCK = 1 << 20


def _features_torch(g, n, dev):
    import torch
    f64 = torch.float64
    tpc_vals = torch.tensor([32, 64, 128, 192, 256, 512, 1024], dtype=f64, device=dev)
    probs = torch.tensor([.05, .15, .30, .05, .30, .10, .05], dtype=f64, device=dev)
    tpc = tpc_vals[torch.multinomial(probs, n, replacement=True, generator=g)]
    U = lambda lo, hi: torch.rand(n, dtype=f64, device=dev, generator=g) * (hi - lo) + lo
    ctas = torch.clamp(torch.round(10.0 ** U(0.0, 5.5)), min=1.0)
    per_thread = 10.0 ** U(1.0, 4.5)
    alpha = torch.tensor([4.0, 2.0, 2.0, 0.5, 0.5, 3.0], dtype=f64, device=dev).expand(n, 6)
    gam = torch._standard_gamma(alpha.contiguous(), generator=g)
    mix = gam / gam.sum(1, keepdim=True)
    total = per_thread * tpc * ctas
    cls = torch.round(mix * total[:, None])
    arith, logic, control, special, sync, mem = (cls[:, i] for i in range(6))
    vsz = torch.tensor([4.0, 8.0, 16.0], dtype=f64, device=dev)[torch.randint(0, 3, (n,), device=dev, generator=g)]
    gvol = torch.round(mem * vsz * U(0.3, 1.0))
    pvol = torch.round(10.0 ** U(1.0, 3.0) * tpc * ctas)
    svol = torch.round(mem * 4.0 * U(0.0, 0.7))
    ai = arith / torch.clamp(gvol, min=1.0)
    tot = arith + logic + control + special + sync + mem
    X = torch.stack([tpc, ctas, tot, special, logic, control, arith, sync, gvol, pvol, svol, ai], dim=1)
    return X, dict(arith=arith, special=special, mem=mem, gvol=gvol, tpc=tpc, ctas=ctas, sync=sync, total=tot)


def scaled_device(n: int, p: int = 64, seed: int = SEED, device="cuda", with_y: bool = True):
    """scaled() on the GPU (torch tensors [n, p] fp64 and [n] fp64 > 0, K20 time target):
    paper features, per-class sub-counts, 4 low-cardinality columns."""
    import torch
    assert p >= 16
    dev = torch.device(device)
    X = torch.empty((n, p), dtype=torch.float64, device=dev)
    y = torch.empty(n, dtype=torch.float64, device=dev) if with_y else None
    g = torch.Generator(device=dev)
    k20 = GPUS["K20"]
    lanes = k20["sms"] * 64.0 * k20["clk"] * 1e6
    nsub = p - 12 - 4
    for b0 in range(0, n, DEV_BLOCK):
        m = min(DEV_BLOCK, n - b0)
        g.manual_seed((seed * 1000003 + 7 * p + b0 // DEV_BLOCK) & 0x7FFFFFFFFFFFFFFF)
        X12, parts = _features_torch(g, m, dev)
        blk = X[b0:b0 + m]
        blk[:, :12] = X12
        cls = torch.stack([X12[:, 6], X12[:, 4], X12[:, 5], X12[:, 3]], dim=1)
        fr = torch.rand((m, nsub), dtype=torch.float64, device=dev, generator=g) * 0.45 + 0.05
        idx = torch.arange(nsub, device=dev) % 4
        blk[:, 12:12 + nsub] = torch.round(cls[:, idx] * fr)
        blk[:, 12 + nsub:] = torch.randint(0, 8, (m, 4), device=dev, generator=g).to(torch.float64)
        if with_y:
            comp = (parts["arith"] + 4.0 * parts["special"] + parts["total"] * 0.25) / lanes * 1e6
            memt = parts["gvol"] / (k20["bw"] * 1e9) * 1e6
            sync = parts["sync"] / lanes * 1e6 * 8.0
            t = 2.0 + comp + memt + sync
            y[b0:b0 + m] = t * torch.exp(torch.randn(m, dtype=torch.float64, device=dev, generator=g) * k20["sigma"])
    return (X, y) if with_y else X


def queries_device(n: int, p: int = 64, seed: int = SEED, device="cuda"):
    """Held-out query rows for inference on the GPU (seed + 1, as queries())."""
    return scaled_device(n, p, seed + 1, device, with_y=False)
