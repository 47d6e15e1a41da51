"""Star-phylogeny protein-family generator (SURVEY.md §8(d) "Synthetic inputs").

Recipe (fixed here; DESIGN.md §3 restates it):

* alphabet of 20 residues, codes 0..19 standing for ``ACDEFGHIKLMNPQRSTVWY``;
* ``families`` families of ``n // families`` members each;
* each family has one uniform random ancestor; its length is U{lo..hi} inclusive,
  or (config 4) ``round(lognormal(ln(mean) - sigma^2/2, sigma))`` clipped to
  ``[lo, hi]`` so the pre-clip mean is ``mean``;
* every member is mutated independently from its ancestor (star phylogeny):
  - substitution: each site with probability ``p_sub`` becomes a uniform
    *different* residue;
  - indels: one left-to-right pass over the substituted sites; at each site an
    event happens with probability ``p_indel``: insertion or deletion with 1/2
    each, length U{1,2,3}.  An insertion emits the site and then the inserted
    uniform residues; a deletion removes that site and the following ones, ``len``
    sites in total.  Events on deleted sites are ignored.
  - a member shorter than ``min_len`` (3 = k) is redrawn (never expected);
* a final ``rng.permutation(n)`` shuffles members so families interleave;
* RNG: ``numpy.random.Generator(PCG64(seed))``, seed = config index 1..5.

The output is a CSR: ``residues`` (uint8, concatenated), ``offsets`` (int64,
n+1) and ``family`` (int32, n).  ``sha256`` covers residues and offsets.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

ALPHABET = "ACDEFGHIKLMNPQRSTVWY"


@dataclass(frozen=True)
class WorkloadConfig:
    """One BASELINE.json config (``configs[i]``) plus the partition parameters."""

    name: str
    n: int
    families: int
    length: tuple  # ("uniform", lo, hi) or ("lognormal", mean, sigma, lo, hi)
    p_sub: float
    p_indel: float
    p: int                   # buckets = logical blocks
    samples_per_block: int   # k_b, BJ "regular samples per bucket"
    seed: int
    k: int = 3
    alphabet: int = 20


CONFIGS = {
    1: WorkloadConfig("cfg1", 200, 8, ("uniform", 100, 400), 0.30, 0.05, 4, 16, 1),
    2: WorkloadConfig("cfg2", 2000, 40, ("uniform", 200, 400), 0.25, 0.05, 8, 64, 2),
    3: WorkloadConfig("cfg3", 20000, 200, ("uniform", 200, 500), 0.30, 0.05, 8, 128, 3),
    4: WorkloadConfig("cfg4", 100000, 1000, ("lognormal", 350.0, 0.4, 50, 2000), 0.35, 0.08, 8, 256, 4),
    5: WorkloadConfig("cfg5", 5000, 50, ("uniform", 1000, 5000), 0.20, 0.03, 8, 64, 5),
}


@dataclass
class Dataset:
    residues: np.ndarray          # uint8 [sum n_i]
    offsets: np.ndarray           # int64 [n+1]
    family: np.ndarray            # int32 [n]
    config: WorkloadConfig | None = None
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.offsets.shape[0] - 1)

    def lengths(self) -> np.ndarray:
        return np.diff(self.offsets)

    def seq(self, i: int) -> np.ndarray:
        return self.residues[self.offsets[i]:self.offsets[i + 1]]

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(self.residues).tobytes())
        h.update(np.ascontiguousarray(self.offsets).astype("<i8").tobytes())
        return h.hexdigest()

    def subset(self, idx) -> "Dataset":
        """CSR of the sequences ``idx`` (in that order)."""
        idx = np.asarray(idx, dtype=np.int64)
        lens = self.lengths()[idx]
        offs = np.zeros(idx.shape[0] + 1, dtype=np.int64)
        np.cumsum(lens, out=offs[1:])
        res = np.empty(int(offs[-1]), dtype=np.uint8)
        for j, i in enumerate(idx):
            res[offs[j]:offs[j + 1]] = self.seq(int(i))
        return Dataset(res, offs, self.family[idx].copy(), self.config)


def from_sequences(seqs, family=None) -> Dataset:
    """CSR from a list of code arrays (or strings over ``ALPHABET``)."""
    arrs = []
    for s in seqs:
        if isinstance(s, str):
            arrs.append(np.array([ALPHABET.index(c) for c in s], dtype=np.uint8))
        else:
            arrs.append(np.asarray(s, dtype=np.uint8))
    offs = np.zeros(len(arrs) + 1, dtype=np.int64)
    np.cumsum([a.shape[0] for a in arrs], out=offs[1:])
    res = np.concatenate(arrs) if arrs else np.zeros(0, dtype=np.uint8)
    fam = np.zeros(len(arrs), dtype=np.int32) if family is None else np.asarray(family, dtype=np.int32)
    return Dataset(res.astype(np.uint8), offs, fam)


def _ancestor_length(rng, spec) -> int:
    if spec[0] == "uniform":
        _, lo, hi = spec
        return int(rng.integers(lo, hi + 1))
    _, mean, sigma, lo, hi = spec
    mu = np.log(mean) - sigma * sigma / 2.0
    return int(min(max(int(round(rng.lognormal(mu, sigma))), lo), hi))


def _mutate(rng, anc: np.ndarray, p_sub: float, p_indel: float, alphabet: int) -> np.ndarray:
    L = anc.shape[0]
    sub = rng.random(L) < p_sub
    shift = rng.integers(1, alphabet, size=L)
    x = np.where(sub, (anc.astype(np.int64) + shift) % alphabet, anc).astype(np.uint8)
    ev = np.flatnonzero(rng.random(L) < p_indel)
    if ev.shape[0] == 0:
        return x
    is_ins = rng.random(ev.shape[0]) < 0.5
    lens = rng.integers(1, 4, size=ev.shape[0])
    ins_res = rng.integers(0, alphabet, size=int(lens.sum())).astype(np.uint8)
    parts = []
    pos = 0
    ins_pos = 0
    for e in range(ev.shape[0]):
        u = int(ev[e])
        ln = int(lens[e])
        if u < pos:            # site already deleted
            if is_ins[e]:
                ins_pos += ln
            continue
        if is_ins[e]:
            parts.append(x[pos:u + 1])
            parts.append(ins_res[ins_pos:ins_pos + ln])
            ins_pos += ln
            pos = u + 1
        else:
            parts.append(x[pos:u])
            pos = min(u + ln, L)
    parts.append(x[pos:])
    return np.concatenate(parts)


def generate(cfg: WorkloadConfig, min_len: int | None = None) -> Dataset:
    """Generate the workload ``cfg`` deterministically from ``cfg.seed``."""
    min_len = cfg.k if min_len is None else min_len
    rng = np.random.Generator(np.random.PCG64(cfg.seed))
    per = cfg.n // cfg.families
    assert per * cfg.families == cfg.n, "n must be a multiple of families"
    seqs = []
    fam = np.empty(cfg.n, dtype=np.int32)
    for f in range(cfg.families):
        L = _ancestor_length(rng, cfg.length)
        anc = rng.integers(0, cfg.alphabet, size=L).astype(np.uint8)
        for m in range(per):
            while True:
                s = _mutate(rng, anc, cfg.p_sub, cfg.p_indel, cfg.alphabet)
                if s.shape[0] >= min_len:
                    break
            fam[f * per + m] = f
            seqs.append(s)
    perm = rng.permutation(cfg.n)
    lens = np.array([seqs[i].shape[0] for i in perm], dtype=np.int64)
    offs = np.zeros(cfg.n + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    res = np.concatenate([seqs[i] for i in perm]).astype(np.uint8)
    ds = Dataset(res, offs, fam[perm].copy(), cfg)
    ds.meta = {"config": cfg.name, "seed": cfg.seed, "n": cfg.n, "residues": int(offs[-1]),
               "max_len": int(lens.max()), "min_len": int(lens.min()), "sha256": ds.sha256()}
    return ds


def generate_config(idx: int) -> Dataset:
    return generate(CONFIGS[idx])


def random_codes(rng: np.random.Generator, n: int, alphabet: int = 20) -> np.ndarray:
    """Uniform residue codes (helper for small seeded test inputs)."""
    return rng.integers(0, alphabet, size=n).astype(np.uint8)
