"""Seeded synthetic workloads shared by the oracle side (tests/, bench cpu leg)
and the product side (bench.py, smoke()).

This module holds NONE of the method's arithmetic: it only describes problem
instances (patch grid, spline degree, elements per patch, per-patch material
arrays, time grid, source kind) and draws the seeded random material values.
Both `oracle/` and `paper_2510_23446_b200/` receive these arrays as plain
inputs; neither imports the other.

Configs follow /root/repo/BASELINE.json `configs` (restated in SURVEY.md §8(d)
table "Cfg 1..5"); readings of the gaps (A(0)=0, T=1, seed 0, draw order,
central column, cluster growth rule) are SURVEY.md §8(c) Q11 and DESIGN.md §3.
"""
from __future__ import annotations

from dataclasses import dataclass, field, asdict
from typing import List, Tuple

import numpy as np

# source kinds (shared vocabulary with include/tcg_ietidp.h TCG_SOURCE_*)
SOURCE_NONE = 0
SOURCE_CURL_PSI = 1   # J = curl(0,0,sin(pi x)sin(pi y)sin(pi z)) * sin(2 pi t)   (BJ configs)
SOURCE_MMS = 2        # J = [2 pi^2 nu (1-e^-t) + sigma e^-t] S(x), S=(sy sz, sx sz, sx sy)
SOURCE_PAPER = 3      # the paper's A = e^-t (sx cy cz, -2 cx sy cz, cx cy sz), inhomogeneous Dirichlet


@dataclass
class Problem:
    name: str
    npatch: Tuple[int, int, int]
    lo: Tuple[float, float, float]
    hi: Tuple[float, float, float]
    p: int
    elems: Tuple[int, int, int]          # elements per patch per direction
    sigma: np.ndarray                    # (P,) >= 0, patch id = ix + Px*(iy + Py*iz)
    nu: np.ndarray                       # (P,) > 0
    T: float = 1.0
    n_steps: int = 10
    source: int = SOURCE_CURL_PSI
    source_params: tuple = ()            # kind 1: (amp, freq) default (1, 1); kind 2: (amp,) default (1,)
    rtol: float = 1e-10
    max_iter: int = 5000
    scaling: int = 1                     # 0 = none (paper P:L170), 1 = rho (BJ.ns "scaled")
    tree_order: int = 0                  # 0 ascending ids within a rank, 1 descending
    warm_start: int = 0                  # 0: lambda0 = 0 (paper); k: projection on the last k solutions
    track_errors: bool = False           # source 3: accumulate eps_B, eps_E every step
    nl: np.ndarray = None                # (P, 3) Brauer parameters (k1, k2, k3) per patch, nu = k1 exp(k2 |B|^2) + k3;
                                         # all-zero rows (or None) = linear patch with nu_s (R25)
    newton_tol: float = 1e-8             # Newton stop: ||a_{k+1} - a_k|| <= newton_tol ||a_{k+1}|| (per-patch vectors)
    newton_max: int = 20
    extra: dict = field(default_factory=dict)

    @property
    def n_patches(self) -> int:
        return int(np.prod(self.npatch))

    @property
    def dt(self) -> float:
        return self.T / self.n_steps

    def describe(self) -> dict:
        d = asdict(self)
        d["sigma"] = [float(x) for x in self.sigma]
        d["nu"] = [float(x) for x in self.nu]
        d["nl"] = None if self.nl is None else [[float(v) for v in row] for row in self.nl]
        return d


def patch_index(ix: int, iy: int, iz: int, npatch) -> int:
    return ix + npatch[0] * (iy + npatch[1] * iz)


def patch_coords(pid: int, npatch) -> Tuple[int, int, int]:
    ix = pid % npatch[0]
    iy = (pid // npatch[0]) % npatch[1]
    iz = pid // (npatch[0] * npatch[1])
    return ix, iy, iz


def _grid(npatch):
    return [(ix, iy, iz) for iz in range(npatch[2]) for iy in range(npatch[1]) for ix in range(npatch[0])]


def cfg1() -> Problem:
    """BJ configs[0]: 2x2x2 cubes of (0,1)^3, p=2, 2 el/patch/dir, conductor z<0.5 (sigma=1), nu=1, 10 steps."""
    npatch = (2, 2, 2)
    sig = np.array([1.0 if iz == 0 else 0.0 for (_, _, iz) in _grid(npatch)])
    return Problem("cfg1", npatch, (0, 0, 0), (1, 1, 1), 2, (2, 2, 2), sig, np.ones(8), 1.0, 10)


def cfg2() -> Problem:
    """BJ configs[1]: 4x4x4, p=2, 4 el/patch/dir, conductor = central 2x2x2 block (sigma=1e3), nu=1, 50 steps."""
    npatch = (4, 4, 4)
    sig = np.array([1e3 if (ix in (1, 2) and iy in (1, 2) and iz in (1, 2)) else 0.0
                    for (ix, iy, iz) in _grid(npatch)])
    return Problem("cfg2", npatch, (0, 0, 0), (1, 1, 1), 2, (4, 4, 4), sig, np.ones(64), 1.0, 50)


def cfg3(seed: int = 0) -> Problem:
    """BJ configs[2]: 4x4x4, p=3, 8 el/patch/dir, conductor z<0.5 (sigma=1e6),
    nu = 10^U(-3,0) per patch (64 draws in patch-id order, PCG64 seed 0), 50 steps."""
    npatch = (4, 4, 4)
    rng = np.random.default_rng(seed)
    nu = 10.0 ** rng.uniform(-3.0, 0.0, size=64)
    sig = np.array([1e6 if iz in (0, 1) else 0.0 for (_, _, iz) in _grid(npatch)])
    return Problem("cfg3", npatch, (0, 0, 0), (1, 1, 1), 3, (8, 8, 8), sig, nu, 1.0, 50)


def _euler_char_and_complement_ok(cells: set, npatch) -> Tuple[int, bool]:
    """Euler characteristic of the closed union of unit cubes, and whether the
    complement cells (inside the patch box) are face-connected."""
    V, E, F = set(), set(), set()
    for (x, y, z) in cells:
        for dx in (0, 1):
            for dy in (0, 1):
                for dz in (0, 1):
                    V.add((x + dx, y + dy, z + dz))
        for a in (0, 1):
            for b in (0, 1):
                E.add((0, x, y + a, z + b))
                E.add((1, x + a, y, z + b))
                E.add((2, x + a, y + b, z))
        for a in (0, 1):
            F.add((0, x + a, y, z))
            F.add((1, x, y + a, z))
            F.add((2, x, y, z + a))
    chi = len(V) - len(E) + len(F) - len(cells)
    comp = [c for c in _grid(npatch) if c not in cells]
    if not comp:
        return chi, True
    comp_set = set(comp)
    seen = {comp[0]}
    stack = [comp[0]]
    while stack:
        x, y, z = stack.pop()
        for d in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
            nb = (x + d[0], y + d[1], z + d[2])
            if nb in comp_set and nb not in seen:
                seen.add(nb)
                stack.append(nb)
    return chi, len(seen) == len(comp)


def grow_cluster(npatch, start, size, rng) -> List[int]:
    """SURVEY §8(d) 'cfg4 cluster growth': frontier = sorted ids of face neighbours
    not in the cluster; draw rng.integers(len(frontier)); accept iff chi == 1 and the
    insulator cells stay face-connected; otherwise drop that candidate and redraw."""
    cells = {tuple(start)}
    while len(cells) < size:
        frontier = set()
        for (x, y, z) in cells:
            for d in ((1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)):
                nb = (x + d[0], y + d[1], z + d[2])
                if all(0 <= nb[i] < npatch[i] for i in range(3)) and nb not in cells:
                    frontier.add(nb)
        cand = sorted(frontier, key=lambda c: patch_index(*c, npatch))
        while cand:
            k = int(rng.integers(len(cand)))
            c = cand.pop(k)
            trial = cells | {c}
            chi, ok = _euler_char_and_complement_ok(trial, npatch)
            if chi == 1 and ok:
                cells = trial
                break
        else:
            raise RuntimeError("cluster growth stalled")
    return sorted(patch_index(*c, npatch) for c in cells)


def cfg4(seed: int = 0) -> Problem:
    """BJ configs[3]: 8x8x8, p=2, 6 el/patch/dir; 128-patch conductor cluster grown from
    (3,3,3); sigma = 10^U(3,7) over conductors in patch-id order, then nu = 10^U(-3,0) for
    all 512 patches; 100 steps."""
    npatch = (8, 8, 8)
    rng = np.random.default_rng(seed)
    cluster = grow_cluster(npatch, (3, 3, 3), 128, rng)
    sig = np.zeros(512)
    sig[cluster] = 10.0 ** rng.uniform(3.0, 7.0, size=len(cluster))
    nu = 10.0 ** rng.uniform(-3.0, 0.0, size=512)
    pr = Problem("cfg4", npatch, (0, 0, 0), (1, 1, 1), 2, (6, 6, 6), sig, nu, 1.0, 100)
    pr.extra["cluster"] = cluster
    return pr


def cfg5() -> Problem:
    """BJ configs[4]: (0,2)x(0,2)x(0,1) as 16x16x8 patches, p=3, 6 el/patch/dir; conductor
    z<0.5 (iz in 0..3, sigma=1e6); nu=1e-3 on the central column ix,iy in 6..9, else 1; 100 steps."""
    npatch = (16, 16, 8)
    sig = np.array([1e6 if iz <= 3 else 0.0 for (_, _, iz) in _grid(npatch)])
    nu = np.array([1e-3 if (6 <= ix <= 9 and 6 <= iy <= 9) else 1.0 for (ix, iy, _) in _grid(npatch)])
    return Problem("cfg5", npatch, (0, 0, 0), (2, 2, 1), 3, (6, 6, 6), sig, nu, 1.0, 100)


def paper(p: int, divs: int, n_steps: int, T: float = 1.0) -> Problem:
    """The paper's experiment: Omega = (0,1)^3 split at x = 1/2 into two patches,
    conductor x < 1/2 (sigma = 1) and insulator (sigma = 0), nu = 1 in both; `divs` elements per
    direction over the whole cube (divs/2 along x per patch); A = e^-t S prescribed (source 3,
    inhomogeneous Dirichlet lifting, A(0) from the same projection); PCG "without scaling"
     and tolerance 1e-6."""
    if divs % 2:
        raise ValueError("divs must be even (two patches along x)")
    pr = Problem(f"paper-p{p}-d{divs}-nt{n_steps}", (2, 1, 1), (0, 0, 0), (1, 1, 1), p, (divs // 2, divs, divs),
                 np.array([1.0, 0.0]), np.array([1.0, 1.0]), T, n_steps, SOURCE_PAPER, rtol=1e-6, scaling=0)
    pr.track_errors = True
    return pr


# Brauer parameters of the nonlinear workloads (R25): nu(0) = k1 + k3 = 1, nu grows
# to ~2.7 at |B| = 0.5 and ~55 at |B| = 1 (the unit-amplitude BJ source gives |B| up to ~0.5)
NL_SOFT = (0.1, 4.0, 0.9)


def nonlinear(base: Problem, patches, k=NL_SOFT, amp: float = 1.0, name: str | None = None, **kw) -> Problem:
    """`base` with Brauer reluctivity k on the listed patches, source
    amplitude amp (kind 1 params (amp, 1)); other fields of `base` kept."""
    P = base.n_patches
    nl = np.zeros((P, 3))
    for s in patches:
        nl[s] = k
    base.nl = nl
    base.source_params = (float(amp), 1.0)
    base.name = name or f"{base.name}-nl"
    for key, v in kw.items():
        setattr(base, key, v)
    return base


def nl1() -> Problem:
    """cfg1 with its 4 conductor patches nonlinear (NL_SOFT), source amplitude 3."""
    b = cfg1()
    return nonlinear(b, [s for s in range(b.n_patches) if b.sigma[s] > 0], amp=3.0, name="nl1")


def nl2() -> Problem:
    """cfg2 with the conductor block and the ring of insulator patches around it in x,y
    nonlinear (NL_SOFT), source amplitude 3, 50 steps."""
    b = cfg2()
    sel = [s for s, (ix, iy, iz) in enumerate(_grid(b.npatch)) if iz in (1, 2)]
    return nonlinear(b, sel, amp=3.0, name="nl2")


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5, "nl1": nl1, "nl2": nl2}


def get(name: str) -> Problem:
    return CONFIGS[name]()


def custom(npatch, p, elems, sigma, nu, lo=(0, 0, 0), hi=(1, 1, 1), n_steps=4, T=1.0,
           source=SOURCE_CURL_PSI, name="custom", **kw) -> Problem:
    P = int(np.prod(npatch))
    sigma = np.broadcast_to(np.asarray(sigma, dtype=np.float64), (P,)).copy()
    nu = np.broadcast_to(np.asarray(nu, dtype=np.float64), (P,)).copy()
    return Problem(name, tuple(npatch), tuple(lo), tuple(hi), p, tuple(elems), sigma, nu, T, n_steps,
                   source, **kw)
