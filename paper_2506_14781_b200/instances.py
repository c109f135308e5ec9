"""Host-side instance construction for the 2D-PT sweep engine.

Synthetic generators for the BASELINE.json configurations (there is no public
benchmark suite) plus the reference's copy-chain sparsifier and
the canonical colour order the engine sweeps in.

* ``sparsify`` restates ``tempergrid::sparsify``
  (/root/reference/proj/src/constraints.cpp:50-120): copies ``u*c+k`` joined in
  a chain, each logical edge placed on the copy with the most remaining
  degree budget (first wins ties), fields on the first copy.
* ``five_node_complete`` is the reference's default toy instance
  (src/instances.cpp:47-67).
* ``wishart_planted`` follows the planted-Wishart construction of
  src/instances.cpp:12-45 (columns projected orthogonal to the planted state,
  rescaled by sqrt(n/(n-1)), J = -(W W^T)/n) with the all-ones planted state
  of BASELINE.json (gauge-equivalent) and couplings
  rounded to float32 (config 2-4 are float32 instances).
* ``k10_pm1`` (config 1), ``bipartite_3regular`` (config 5) are new generators
  described in SURVEY.md §8d.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np


class ConfigError(ValueError):
    """Bad user input (reference ``config_error``, CLI exit code 2)."""


class ResourceError(RuntimeError):
    """Request beyond a resource guard (reference ``resource_error``, exit 3)."""


@dataclass
class Problem:
    """A ConstrainedProblem in plain arrays: cost couplings (i, j, w), fields,
    and chain-constraint pairs (a, b).  Mirrors ``ConstrainedProblem``
    (/root/reference/proj/include/tempergrid/constraints.hpp:44-48)."""

    n: int
    ci: np.ndarray
    cj: np.ndarray
    cw: np.ndarray
    fields: np.ndarray
    pa: np.ndarray
    pb: np.ndarray
    copies: Optional[List[List[int]]] = None  # sparsification map (logical -> chain)
    meta: dict = field(default_factory=dict)

    @staticmethod
    def make(n: int, couplings: Sequence[Tuple[int, int, float]], fields: Sequence[float],
             pairs: Sequence[Tuple[int, int]] = ()) -> "Problem":
        c = np.asarray(couplings, dtype=np.float64).reshape(-1, 3)
        p = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
        return Problem(
            n=int(n),
            ci=c[:, 0].astype(np.int32), cj=c[:, 1].astype(np.int32),
            cw=np.ascontiguousarray(c[:, 2]),
            fields=np.asarray(fields, dtype=np.float64).copy(),
            pa=p[:, 0].astype(np.int32).copy(), pb=p[:, 1].astype(np.int32).copy())

    @property
    def n_couplings(self) -> int:
        return int(self.ci.shape[0])

    @property
    def n_pairs(self) -> int:
        return int(self.pa.shape[0])

    def permuted(self, order: np.ndarray) -> "Problem":
        """Relabel so that new index k is old spin ``order[k]``."""
        inv = np.empty(self.n, dtype=np.int64)
        inv[np.asarray(order)] = np.arange(self.n)
        copies = None
        if self.copies is not None:
            copies = [[int(inv[p]) for p in chain] for chain in self.copies]
        return Problem(self.n, inv[self.ci].astype(np.int32), inv[self.cj].astype(np.int32),
                       self.cw.copy(), self.fields[np.asarray(order)].copy(),
                       inv[self.pa].astype(np.int32), inv[self.pb].astype(np.int32),
                       copies, dict(self.meta))


# --------------------------------------------------------------- sparsify

def sparsify(n: int, couplings: Sequence[Tuple[int, int, float]], fields: Sequence[float],
             copies_per_node: int, max_degree: int) -> Problem:
    """Restates constraints.cpp:50-120 (see module docstring)."""
    if copies_per_node < 1:
        raise ConfigError("sparsify: copies_per_node must be >= 1")
    # IsingModel canonical order: i<j, sorted (ising.cpp:29-41)
    canon = sorted(((min(i, j), max(i, j), float(w)) for i, j, w in couplings))
    if copies_per_node == 1:
        pr = Problem.make(n, canon, fields, [])
        pr.copies = [[u] for u in range(n)]
        return pr
    if max_degree < 3:
        raise ConfigError("sparsify: max_degree must be >= 3 with copy chains")
    c = copies_per_node
    chain_deg = [1 if (k == 0 or k == c - 1) else 2 for k in range(c)]
    budget = [[max_degree - chain_deg[k] for k in range(c)] for _ in range(n)]

    def place(u: int) -> int:
        best = -1
        for k in range(c):
            if best < 0 or budget[u][k] > budget[u][best]:
                best = k
        if budget[u][best] <= 0:
            raise ConfigError(f"sparsify: degree cap {max_degree} too small for node {u}")
        budget[u][best] -= 1
        return u * c + best

    phys = []
    for i, j, w in canon:
        pu = place(i)
        pv = place(j)
        phys.append((pu, pv, w))
    f = [0.0] * (n * c)
    for u in range(n):
        f[u * c] = float(fields[u])
    pairs = [(u * c + k, u * c + k + 1) for u in range(n) for k in range(c - 1)]
    pr = Problem.make(n * c, phys, f, pairs)
    pr.copies = [[u * c + k for k in range(c)] for u in range(n)]
    deg = np.zeros(n * c, dtype=np.int64)
    np.add.at(deg, pr.ci, 1)
    np.add.at(deg, pr.cj, 1)
    np.add.at(deg, pr.pa, 1)
    np.add.at(deg, pr.pb, 1)
    if deg.max(initial=0) > max_degree:
        raise ConfigError("sparsify: degree cap violated at physical spin %d" % int(deg.argmax()))
    return pr


def min_copies(n_logical_degree: int, max_degree: int) -> int:
    """Smallest chain length c with capacity c*(D-2)+2 >= degree (constraints.cpp:71-95)."""
    c = 1
    while c * (max_degree - 2) + 2 < n_logical_degree:
        c += 1
    return c


# ----------------------------------------------------------- colour order

# False: never load the engine library for instance construction (bench.py's
# reference arm must not map libtempergrid_b200.so; set TG_INSTANCES_PY=1 or
# call use_native_helpers(False)).
_NATIVE_HELPERS = os.environ.get("TG_INSTANCES_PY", "0") in ("", "0")


def use_native_helpers(on: bool) -> None:
    global _NATIVE_HELPERS
    _NATIVE_HELPERS = bool(on)


def canonical_order(pr: Problem) -> Tuple[np.ndarray, np.ndarray, int]:
    """Greedy index-order colouring of cost+chain edges, then a stable sort by
    (colour, chain degree, cost degree).  Returns (order, colour, n_colours).
    Uses the engine library's host helper (tg_canonical_order) when it is
    built and allowed, else the pure-Python restatement below; tests check
    they agree."""
    if _NATIVE_HELPERS:
        try:
            return canonical_order_native(pr)
        except Exception:  # noqa: BLE001 - library not built: host-only path
            pass
    return canonical_order_py(pr)


def canonical_order_native(pr: Problem) -> Tuple[np.ndarray, np.ndarray, int]:
    import ctypes as C
    from . import _lib
    L = _lib.lib()
    arrs = [np.ascontiguousarray(a, dtype=np.int32) for a in (pr.ci, pr.cj, pr.pa, pr.pb)]
    order = np.zeros(pr.n, np.int32)
    color = np.zeros(pr.n, np.int32)
    nc = C.c_int32()
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    rc = L.tg_canonical_order(pr.n, len(arrs[0]), P(arrs[0]), P(arrs[1]), len(arrs[2]), P(arrs[2]),
                              P(arrs[3]), P(order), P(color), C.byref(nc))
    if rc != 0:
        raise ConfigError("canonical_order: invalid problem")
    return order.astype(np.int64), color.astype(np.int64), int(nc.value)


def canonical_order_py(pr: Problem) -> Tuple[np.ndarray, np.ndarray, int]:
    n = pr.n
    adj: List[List[int]] = [[] for _ in range(n)]
    dc = np.zeros(n, dtype=np.int64)
    dq = np.zeros(n, dtype=np.int64)
    for a, b in zip(pr.ci.tolist(), pr.cj.tolist()):
        adj[a].append(b); adj[b].append(a); dc[a] += 1; dc[b] += 1
    for a, b in zip(pr.pa.tolist(), pr.pb.tolist()):
        adj[a].append(b); adj[b].append(a); dq[a] += 1; dq[b] += 1
    color = np.zeros(n, dtype=np.int64)
    for i in range(n):
        used = {int(color[j]) for j in adj[i] if j < i}
        c = 0
        while c in used:
            c += 1
        color[i] = c
    key = color * (1 << 40) + dq * (1 << 20) + dc
    order = np.argsort(key, kind="stable")
    return order.astype(np.int64), color, int(color.max(initial=-1) + 1)


def to_canonical(pr: Problem) -> Problem:
    order, _, nc = canonical_order(pr)
    out = pr.permuted(order)
    out.meta["n_colors"] = nc
    return out


# ------------------------------------------------------------- generators

def five_node_complete() -> Problem:
    """instances.cpp:55-66"""
    return Problem.make(5, [(0, 1, -1.0), (0, 2, -1.0), (0, 3, -2.0), (0, 4, -2.0),
                            (1, 2, -1.0), (1, 3, -1.0), (1, 4, -2.0), (2, 3, -1.0),
                            (2, 4, -1.0), (3, 4, -2.0)], [0.5, -1.0, 0.5, 0.5, -1.0])


def k10_pm1(seed: int = 1, n: int = 10, copies: int = 2, max_degree: int = 6) -> Problem:
    """Config 1: logical K_n with J_ij = +-1 (fair coin), h = 0, sparsified to
    copy chains (c=2, D=6 -> 20 physical spins)."""
    rng = np.random.default_rng(seed)
    cpl = [(i, j, float(rng.choice([-1.0, 1.0]))) for i in range(n) for j in range(i + 1, n)]
    pr = sparsify(n, cpl, [0.0] * n, copies, max_degree)
    pr.meta.update(kind="k10_pm1", seed=seed, logical=(n, cpl, [0.0] * n))
    return to_canonical(pr)


def wishart_planted(n: int, alpha: float, seed: int, max_degree: int = 3,
                    copies: Optional[int] = None) -> Problem:
    """Configs 2-4: planted Wishart (all-ones ground state), float32 couplings,
    sparsified to degree <= max_degree copy chains."""
    m = int(round(alpha * n))
    if n < 3 or m < 1:
        raise ConfigError("wishart: bad size")
    rng = np.random.default_rng(seed)
    t = np.ones(n)
    z = rng.standard_normal((n, m))
    w = np.sqrt(n / (n - 1.0)) * (z - np.outer(t, (t @ z) / n))
    gram = w @ w.T
    jm = (-gram / n).astype(np.float32).astype(np.float64)
    cpl = [(i, j, float(jm[i, j])) for i in range(n) for j in range(i + 1, n)]
    c = copies if copies is not None else min_copies(n - 1, max_degree)
    pr = sparsify(n, cpl, [0.0] * n, c, max_degree)
    e_planted = -float(sum(w_ for _, _, w_ in cpl))
    pr.meta.update(kind="wishart", n_logical=n, alpha=alpha, seed=seed,
                   planted_energy=e_planted, logical=(n, cpl, [0.0] * n),
                   pmax_cfg=2.0 * float(np.abs(jm).sum(axis=1).max()))
    return to_canonical(pr)


def bipartite_3regular(n: int, seed: int = 1, chain_frac: float = 0.1) -> Problem:
    """Config 5: random bipartite 3-regular graph (sides A=[0,n/2), B=[n/2,n),
    union of 3 random perfect matchings, multi-edges rejected), J = +-1 fair,
    h = 0, plus copy-constraint chain pairs on ``chain_frac`` of the nodes
    (random non-adjacent A-B pairs).  Two colours = the two sides."""
    if n % 2 or n < 8:
        raise ConfigError("bipartite_3regular: n must be even and >= 8")
    h = n // 2
    rng = np.random.default_rng(seed)
    nbrs = np.full((h, 3), -1, dtype=np.int64)  # B-side partner (0..h-1) per A node
    for k in range(3):
        while True:
            perm = rng.permutation(h)
            clash = np.zeros(h, dtype=bool)
            for q in range(k):
                clash |= nbrs[:, q] == perm
            bad = np.nonzero(clash)[0]
            tries = 0
            while bad.size and tries < 100:
                # repair by swapping each clashing target with a random other
                for a in bad:
                    b = int(rng.integers(h))
                    perm[a], perm[b] = perm[b], perm[a]
                clash[:] = False
                for q in range(k):
                    clash |= nbrs[:, q] == perm
                bad = np.nonzero(clash)[0]
                tries += 1
            if not bad.size:
                break
        nbrs[:, k] = perm
    ai = np.repeat(np.arange(h), 3)
    bj = nbrs.reshape(-1) + h
    w = rng.choice(np.array([-1.0, 1.0]), size=ai.size)
    # chain pairs on non-adjacent A-B pairs, disjoint endpoints
    n_pairs = int(round(chain_frac * n / 2))
    a_sel = rng.choice(h, size=n_pairs, replace=False)
    b_pool = rng.permutation(h)
    pa, pb, used_b, bi = [], [], set(), 0
    for a in a_sel.tolist():
        while True:
            b = int(b_pool[bi % h]); bi += 1
            if b not in used_b and b not in set(nbrs[a].tolist()):
                break
        used_b.add(b)
        pa.append(a); pb.append(b + h)
    pr = Problem(n, ai.astype(np.int32), bj.astype(np.int32), w.astype(np.float64),
                 np.zeros(n), np.asarray(pa, dtype=np.int32), np.asarray(pb, dtype=np.int32))
    pr.meta.update(kind="bipartite_3regular", seed=seed, chain_frac=chain_frac)
    return to_canonical(pr)


# -------------------------------------------------------------- schedules

def geometric(lo: float, hi: float, k: int) -> np.ndarray:
    if k == 1:
        return np.array([lo])
    return lo * (hi / lo) ** (np.arange(k) / (k - 1))


def linear(lo: float, hi: float, k: int) -> np.ndarray:
    if k == 1:
        return np.array([lo])
    return lo + (hi - lo) * np.arange(k) / (k - 1)


def dyadic(v: np.ndarray, bits: int = 6) -> np.ndarray:
    """Round to multiples of 2^-bits (keeps the reference's FP64 caches exact,
    SURVEY.md §7 hard part 2)."""
    return np.round(np.asarray(v) * (1 << bits)) / (1 << bits)


def config_schedule(name: str) -> Tuple[np.ndarray, np.ndarray]:
    """(betas, penalties) in reference units (P_ref = P_cfg / 4, SURVEY.md
    Appendix A.5) for the BASELINE.json configs."""
    if name == "c1":
        return geometric(0.1, 3.0, 8), dyadic(linear(0.0, 4.0, 8) / 4.0)
    if name == "c5":
        return geometric(0.2, 5.0, 16), dyadic(linear(0.0, 4.0, 16) / 4.0)
    raise ConfigError(f"unknown config schedule {name}")


def wishart_schedule(pr: Problem, n_beta: int = 16, n_pen: int = 8) -> Tuple[np.ndarray, np.ndarray]:
    pmax_ref = pr.meta["pmax_cfg"] / 4.0
    return geometric(0.2, 5.0, n_beta), linear(0.0, pmax_ref, n_pen)
