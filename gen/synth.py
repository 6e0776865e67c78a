"""Deterministic synthetic Tier-1 data shaped like the paper's profiler output.

The paper's measured data (nvprof 6.5 counters of 128 CUDA n-body variants on
a Tesla K20c, §5) is not available, so every workload is a
seeded stand-in with the paper's *structure*:

* a 2^m version lattice per (program, input, run) group -- "all possible
  combinations of six source-code optimizations ... 64 different versions"
  (§3.3); slot t = g*2^m + v, group g = (p*I + i)*R + r;
* raw counters that are non-negative integers, a cycle count and a runtime
  per slot -- the inputs Tier 1 normalises (§2);
* several runs per input ("profiled ... three times") that differ by
  per-run noise ("noise 0.02"), and inputs of different size
  (Table 1) where smaller inputs give noisier vectors.

Generator recipe (restated in DESIGN.md §"Input recipe"):

G1  counter model shared by all programs ("same hardware"): loadings
    A in R^{C x 8}, A_ck ~ N(0, 1/8); base log-rate b_c ~ U(ln 1e-3, ln 1).
G2  per (program p, input i): latent z_{p,i} = z_p + u_{p,i}, z_p ~ N(0, I_8),
    u_{p,i} ~ N(0, 0.3^2 I_8), shifted along factor 0 by 0.3 x the centred log
    problem size ln(bodies*steps) (Table 1) when sizes are given.  Optimization effects D_{p,j} ~ N(0, 0.4^2 I_8) per bit j; an
    optimization *name* shared by several programs (FTZ, RSQRT, or the generic
    O0..O5) gets half of its variance from a component common to those
    programs.  The "small" optimization (FTZ in C2, O0 elsewhere) is scaled by
    0.05, mirroring "FTZ applied by itself had very little impact".
G3  variant latent Z_v = z_{p,i} + sum_{j: bit j of v set} D_{p,j}.
G4  rate_{c} = exp(b_c + (A Z_v)_c + eps_{p,i,v,c} + eta_{p,i,r,v,c});
    eps ~ N(0, 0.05^2) is fixed across runs (variant idiosyncrasy),
    eta ~ N(0, noise^2 * s_i^2) is per run, s_i = sqrt(smallest size / size_i).
G5  ln rt_ms = 3 + q.Z_v + Z_v^T Q Z_v + nu, q ~ N(0, 0.15^2 I_8) and
    symmetric Q_kl ~ N(0, 0.03^2) global, nu ~ N(0, 0.01^2) per run.
    Runtimes are per slot, so every speedup is lattice-consistent.
G6  cycles = round(rt_ms * 7.06e5) (K20c at 0.706 GHz, "0.7 GHz" P:175);
    counters = round(rate * cycles), stored as FP64 integers.
G7  every draw is keyed by (seed, tag, indices) through numpy SeedSequence,
    so any program/input/run can be regenerated on its own.

Nothing here computes rates, speedups, pairs or anything else of the method.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

# Global optimization ids are alphabetical over both programs (SURVEY §8(c) O6,
# tie-break rule of SPEC S:303 "optimization_id ascending").
OPT_NAMES_C2 = ["CONST", "FTZ", "PEEL", "RSQRT", "SHMEM", "SORT", "UNROLL",
                "VOLA", "VOTE", "WARP"]
# Per-program optimization lists (P:120-128 NB, P:130-137 BH); bit j of the
# version mask = j-th optimization of the program in alphabetical order.
BH_OPTS = ["FTZ", "RSQRT", "SORT", "VOLA", "VOTE", "WARP"]
NB_OPTS = ["CONST", "FTZ", "PEEL", "RSQRT", "SHMEM", "UNROLL"]
# Table 1: (bodies, time steps).
TABLE1 = {
    "NB": [(50_000, 2), (100_000, 2), (100_000, 5), (200_000, 5)],
    "BH": [(125_000, 2), (250_000, 2), (250_000, 5), (500_000, 5),
           (500_000, 10), (1_000_000, 10)],
}
K20C_HZ = 7.06e8  # P:175 "0.7 GHz"; cycles per ms = 7.06e5
LATENT = 8


@dataclass
class Dataset:
    """Tier-1 input for a whole version lattice (SURVEY §8(b) sr_dataset)."""
    n_programs: int
    n_inputs: int
    n_runs: int
    n_opt_bits: int
    n_counters: int
    n_opt_ids: int
    counters: np.ndarray      # float64 [N][C], non-negative integers
    cycles: np.ndarray        # float64 [N], > 0
    runtime_ms: np.ndarray    # float64 [N], > 0
    opt_bit: np.ndarray       # int8 [P][O], bit of optimization o in program p, -1 absent
    opt_names: list = field(default_factory=list)
    program_names: list = field(default_factory=list)

    @property
    def n_groups(self) -> int:
        return self.n_programs * self.n_inputs * self.n_runs

    @property
    def n_slots(self) -> int:
        return self.n_groups << self.n_opt_bits


def _rng(seed: int, *keys: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([int(seed)] + [int(k) for k in keys]))


_TAG_HW, _TAG_Z, _TAG_DCOMMON, _TAG_DSPEC, _TAG_EPS, _TAG_ETA, _TAG_NU = range(1, 8)


def generate(*, n_programs: int, n_inputs: int, n_runs: int, n_counters: int,
             seed: int, opt_names: Sequence[str], program_opts: Sequence[Sequence[str]],
             program_names: Optional[Sequence[str]] = None,
             input_sizes: Optional[Sequence[Sequence[tuple]]] = None,
             small_opt: Optional[str] = None, noise: float = 0.02,
             n_opt_bits: int = 6) -> Dataset:
    """Draw one dataset (recipe G1-G7 in the module docstring).

    program_opts[p][j] is the name of the optimization controlled by bit j of
    program p; opt_names is the global id order.  input_sizes[p][i] =
    (bodies, steps) enables the G2 size shift and G4 size-dependent noise.
    """
    P, I, R, C, m = n_programs, n_inputs, n_runs, n_counters, n_opt_bits
    V = 1 << m
    O = len(opt_names)
    name_to_id = {n: k for k, n in enumerate(opt_names)}
    opt_bit = np.full((P, O), -1, dtype=np.int8)
    for p in range(P):
        assert len(program_opts[p]) == m
        for j, nm in enumerate(program_opts[p]):
            opt_bit[p, name_to_id[nm]] = j

    hw = _rng(seed, _TAG_HW)
    A = hw.normal(0.0, np.sqrt(1.0 / LATENT), size=(C, LATENT))
    b = hw.uniform(np.log(1e-3), np.log(1.0), size=C)
    q = hw.normal(0.0, 0.15, size=LATENT)
    Qr = hw.normal(0.0, 0.03, size=(LATENT, LATENT))
    Q = np.triu(Qr) + np.triu(Qr, 1).T

    # shared (per optimization name) component of the effect vectors
    d_common = {nm: _rng(seed, _TAG_DCOMMON, name_to_id[nm]).normal(0.0, 1.0, LATENT)
                for nm in opt_names}
    n_sharing = {nm: sum(nm in po for po in program_opts) for nm in opt_names}

    masks = np.arange(V)
    bits = ((masks[:, None] >> np.arange(m)[None, :]) & 1).astype(np.float64)  # [V][m]

    N = P * I * R * V
    counters = np.empty((N, C), dtype=np.float64)
    cycles = np.empty(N, dtype=np.float64)
    runtime = np.empty(N, dtype=np.float64)

    for p in range(P):
        D = np.empty((m, LATENT))
        for j, nm in enumerate(program_opts[p]):
            spec = _rng(seed, _TAG_DSPEC, p, j).normal(0.0, 1.0, LATENT)
            if n_sharing[nm] > 1:
                d = np.sqrt(0.5) * d_common[nm] + np.sqrt(0.5) * spec
            else:
                d = spec
            scale = 0.4 * (0.05 if nm == small_opt else 1.0)
            D[j] = scale * d
        if input_sizes is not None:
            logs = np.array([np.log(bd * st) for bd, st in input_sizes[p]], dtype=np.float64)
            shifts = 0.3 * (logs - logs.mean())
            sizes = np.array([bd * st for bd, st in input_sizes[p]], dtype=np.float64)
            noise_scale = np.sqrt(sizes.min() / sizes)
        else:
            shifts = np.zeros(I)
            noise_scale = np.ones(I)
        z_prog = _rng(seed, _TAG_Z, p).normal(0.0, 1.0, LATENT)
        for i in range(I):
            z = z_prog + _rng(seed, _TAG_Z, p, i).normal(0.0, 0.3, LATENT)
            z[0] += shifts[i]
            Z = z[None, :] + bits @ D                        # [V][8]   (G3)
            eps = _rng(seed, _TAG_EPS, p, i).normal(0.0, 0.05, size=(V, C))
            base_log_rate = b[None, :] + Z @ A.T + eps         # [V][C]
            quad = np.einsum("vk,kl,vl->v", Z, Q, Z)
            for r in range(R):
                g = (p * I + i) * R + r
                sl = slice(g * V, (g + 1) * V)
                eta = _rng(seed, _TAG_ETA, p, i, r).normal(0.0, noise * noise_scale[i], size=(V, C))
                nu = _rng(seed, _TAG_NU, p, i, r).normal(0.0, 0.01, size=V)
                rt = np.exp(3.0 + Z @ q + quad + nu)                        # (G5)
                cyc = np.maximum(np.rint(rt * (K20C_HZ / 1e3)), 1.0)         # (G6)
                rate = np.exp(base_log_rate + eta)                           # (G4)
                counters[sl] = np.rint(rate * cyc[:, None])
                cycles[sl] = cyc
                runtime[sl] = rt
    return Dataset(P, I, R, m, C, O, counters, cycles, runtime, opt_bit,
                   list(opt_names), list(program_names or [f"P{p}" for p in range(P)]))
