"""Critical-point trajectory verification (the reference's
tracking.py:145-195 ``verify``), with the face predicates on the device.

The positive faces of the original and of the reconstruction, both at the
original's fixed-point scale, come from the analysis kernel's 12-bit
per-anchor face mask (csrc/analyze.cu, the same exact / SoS predicate as
compression); the flipped-face counts fc_t / fc_s are popcounts of the two
masks' XOR, on the device.  The trajectory graph is linked on the host over
the (sparse) crossed faces: every tet of the space-time mesh crossed by a
trajectory has exactly two crossed faces and contributes the edge joining
them (tracking.py:75-141), so components are simple paths or cycles.
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass
from pathlib import Path
from fractions import Fraction
from itertools import combinations

import numpy as np

from .field import FieldSeries, device_range, scale_for, to_device
from .predicates import face_mask_float, mask_to_faces


class TopologyError(AssertionError):
    """A tet with 1 or >= 3 crossed faces: impossible under exact predicates."""


@dataclass(frozen=True)
class VerifyReport:
    cr: float
    psnr: float
    max_abs_err: float
    fc_t: int            # slice faces whose predicate flipped
    fc_s: int            # slab faces whose predicate flipped
    n_traj_orig: int
    n_traj_recon: int
    isomorphic: bool     # identical node AND edge sets

    @property
    def ok(self) -> bool:
        return self.fc_t == 0 and self.fc_s == 0 and self.isomorphic

    def lines(self):
        yield f"fc_t={self.fc_t}"
        yield f"fc_s={self.fc_s}"
        yield f"n_traj_orig={self.n_traj_orig}"
        yield f"n_traj_recon={self.n_traj_recon}"
        yield f"isomorphic={str(self.isomorphic).lower()}"
        yield f"cr={self.cr:.6g}"
        yield f"psnr={self.psnr:.6g}"
        yield f"max_abs_err={self.max_abs_err:.6g}"


# ------------------------------------------------------------ mesh (tets)
# The space-time mesh of mesh.py:27-56: cell (i, j) of frame t splits into
# the triangles (v00, v01, v11) and (v00, v10, v11); the prism over slab
# [t, t+1] of a triangle (a, b, c) (ascending ids) splits into the tets
# (a, b, c, c'), (a, b, b', c'), (a, a', b', c') (primes: one frame up).

def _tets_around(face, H, W, T):
    """Tets of the mesh that contain `face` (found around its first vertex)."""
    hw = H * W
    a = face[0]
    t, r = divmod(a, hw)
    i, j = divmod(r, W)
    fs = set(face)
    for slab in (t - 1, t):
        if not 0 <= slab < T - 1:
            continue
        for ci in range(max(0, i - 1), min(H - 1, i + 1)):
            for cj in range(max(0, j - 1), min(W - 1, j + 1)):
                v00 = slab * hw + ci * W + cj
                for tri in ((v00, v00 + W, v00 + W + 1),
                            (v00, v00 + 1, v00 + W + 1)):
                    p, q, s = tri
                    for tet in ((p, q, s, s + hw), (p, q, q + hw, s + hw),
                                (p, p + hw, q + hw, s + hw)):
                        if fs <= set(tet):
                            yield tet


def _link(faces, H, W, T):
    """(positives, edges, adj, find) of the crossed-face graph: every tet
    around a crossed face contributes the edge joining its two crossed
    faces (tracking.py:75-106)."""
    positives = faces if isinstance(faces, (set, frozenset)) else set(faces)
    edges = set()
    seen = set()
    for f in positives:
        for tet in _tets_around(f, H, W, T):
            if tet in seen:
                continue
            seen.add(tet)
            crossed = [g for g in (tuple(sorted(c)) for c in combinations(tet, 3))
                       if g in positives]
            if len(crossed) != 2:
                raise TopologyError(
                    f"tet {tet} has {len(crossed)} crossed faces (expected 2)")
            edges.add(tuple(sorted(crossed)))
    adj = {f: [] for f in positives}
    parent = {f: f for f in positives}

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for f, g in edges:
        adj[f].append(g)
        adj[g].append(f)
        rf, rg = find(f), find(g)
        if rf != rg:
            parent[rg] = rf
    for f, nb in adj.items():
        if len(nb) > 2:
            raise TopologyError(f"face {f} has degree {len(nb)}")
    return positives, edges, adj, find


def trajectory_graph(faces, H, W, T):
    """(edges, n_components) of the crossed-face graph (tracking.py:75-141)."""
    positives, edges, _, find = _link(faces, H, W, T)
    return frozenset(edges), len({find(f) for f in positives})


def ordered_components(faces, H, W, T):
    """(edges, chains, loops): each component as an ordered face chain,
    components sorted by their first face (tracking.py:108-139).

    A path starts at its smaller endpoint, a closed loop at its smallest
    face, as in the reference.  A loop's direction is the first neighbour in
    its start face's adjacency list, which the reference fills by iterating
    Python sets; `faces` built by predicates.mask_to_faces (the reference's
    insertion order) and the same set operations here reproduce that order,
    so the chains match the reference's exactly (tests/test_track_cpu.py).
    """
    positives, edges, adj, find = _link(faces, H, W, T)
    groups = {}
    for f in sorted(positives):
        groups.setdefault(find(f), []).append(f)
    chains, loops = [], []
    for members in groups.values():
        ends = [f for f in members if len(adj[f]) <= 1]   # members sorted
        is_loop = not ends
        start = ends[0] if ends else members[0]
        chain, prev, cur = [start], None, start
        while True:
            nxt = None
            for g in adj[cur]:
                if g != prev and (g != start or len(chain) > 2):
                    nxt = g
                    break
            if nxt is None or nxt == start:
                break
            chain.append(nxt)
            prev, cur = cur, nxt
        if len(chain) != len(members):
            raise TopologyError("component is not a simple path or cycle")
        chains.append(chain)
        loops.append(is_loop)
    order = sorted(range(len(chains)), key=lambda k: chains[k][0])
    return (frozenset(edges), [chains[k] for k in order],
            [loops[k] for k in order])


def crossing_point(face, fixed, H, W, dx=1.0, dy=1.0, dt=1.0):
    """(x, y, t) of the zero crossing on a positive face: the origin's exact
    rational barycentric coordinates in (u, v) applied to the vertices'
    (j, i, t) (predicates.py:125-135, 304-318).  `fixed` maps a vertex id
    to its fixed-point (u, v)."""
    a, b, c = face
    (ua, va), (ub, vb), (uc, vc) = fixed[a], fixed[b], fixed[c]
    d_ab = ua * vb - va * ub
    d_bc = ub * vc - vb * uc
    d_ca = uc * va - vc * ua
    df = d_ab + d_bc + d_ca
    if df == 0:
        raise TopologyError(f"degenerate positive face {face}")
    hw = H * W
    sx = sy = st = 0
    for w, num in ((a, d_bc), (b, d_ca), (c, d_ab)):
        t, r = divmod(w, hw)
        i, j = divmod(r, W)
        sx += num * j
        sy += num * i
        st += num * t
    return (float(Fraction(sx, df)) * dx, float(Fraction(sy, df)) * dy,
            float(Fraction(st, df)) * dt)


@dataclass
class TrajectoryGraph:
    """tracking.py:44-56."""
    nodes: dict           # face -> (x, y, t) crossing position
    edges: frozenset      # sorted face pairs
    components: list      # ordered face chains
    loops: list           # bool per component

    @property
    def n_components(self) -> int:
        return len(self.components)

    def component_points(self, k: int):
        return [self.nodes[f] for f in self.components[k]]


def trajectories_from_faces(faces, fixed, H, W, T, dx=1.0, dy=1.0,
                            dt=1.0) -> TrajectoryGraph:
    """Host half of extract_trajectories: link `faces` and place their
    crossing points from the vertices' fixed-point values `fixed`."""
    edges, chains, loops = ordered_components(faces, H, W, T)
    nodes = {fc: crossing_point(fc, fixed, H, W, dx, dy, dt) for fc in faces}
    return TrajectoryGraph(nodes=nodes, edges=edges, components=chains,
                           loops=loops)


def extract_trajectories(f: FieldSeries, dx=None, dy=None, dt=None,
                         scale: float | None = None) -> TrajectoryGraph:
    """Critical-point trajectories of `f` (tracking.py:75-141 over
    to_fixed(f)): the positive faces come from the device analysis kernel
    at the automatic fixed-point scale (or `scale`); the fixed-point values
    of their vertices are gathered and rounded on the device; linking and
    the exact crossing points run on the host over that sparse set."""
    import torch
    H, W, T = f.H, f.W, f.T
    dx = f.dx if dx is None else dx
    dy = f.dy if dy is None else dy
    dt = f.dt if dt is None else dt
    du, dv = to_device(f.u), to_device(f.v)
    if scale is None:
        _, _, ma = device_range(du, dv)
        scale = scale_for(ma)
    faces = _positive_faces(face_mask_float(H, W, T, du, dv, scale, host=False),
                            H, W, T)
    ids = sorted({w for fc in faces for w in fc})
    fixed = {}
    if ids:
        idx = torch.as_tensor(ids, dtype=torch.int64, device=du.device)

        def rha(x):   # field.py:295-297, in float64 on the device
            x = x.double() * scale
            return (torch.sign(x) * torch.floor(torch.abs(x) + 0.5)).to(torch.int64)

        fixed = {w: (uu, vv) for w, uu, vv in
                 zip(ids, rha(du[idx]).cpu().tolist(), rha(dv[idx]).cpu().tolist())}
    return trajectories_from_faces(faces, fixed, H, W, T, dx, dy, dt)


def write_trajectory_csv(graph: TrajectoryGraph, path) -> None:
    """component id, ordered crossing points, loop flag (tracking.py:271-280)."""
    with Path(path).open("w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["component", "x", "y", "t", "loop"])
        for k, chain in enumerate(graph.components):
            flag = int(graph.loops[k])
            for fc in chain:
                x, y, t = graph.nodes[fc]
                w.writerow([k, f"{x:.9g}", f"{y:.9g}", f"{t:.9g}", flag])


# ------------------------------------------------------------------ verify

def _popcount12(x):
    """Per-element popcount of the low 12 bits, summed (torch, on device):
    SWAR bit counting in int32, one reduction, one host read."""
    import torch
    v = x & 0xFFF
    v = v - ((v >> 1) & 0x555)
    v = (v & 0x333) + ((v >> 2) & 0x333)
    v = (v + (v >> 4)) & 0x0F0F
    v = (v + (v >> 8)) & 0x1F
    return int(v.sum(dtype=torch.int64).item())


def _positive_faces(mask, H, W, T):
    import torch
    nz = torch.nonzero(mask).flatten()
    anchors = nz.cpu().numpy()
    bits = mask[nz].cpu().numpy().view(np.uint16)
    sparse = np.zeros(H * W * T, np.uint16)
    sparse[anchors] = bits
    sl, sb = mask_to_faces(sparse, H, W, T)
    return sl | sb


def verify(orig: FieldSeries, recon: FieldSeries,
           archive_size: int | None = None,
           scale: float | None = None) -> VerifyReport:
    """Compare predicates and trajectory graphs at a common fixed-point scale
    (tracking.py:170-195); `scale` defaults to the original's automatic
    scale (the one compression used)."""
    import torch
    if (orig.H, orig.W, orig.T) != (recon.H, recon.W, recon.T):
        raise ValueError("dimension mismatch between original and reconstruction")
    H, W, T = orig.H, orig.W, orig.T
    ou, ov = to_device(orig.u), to_device(orig.v)
    ru, rv = to_device(recon.u), to_device(recon.v)
    if scale is None:
        _, _, ma = device_range(ou, ov)
        scale = scale_for(ma)
    m_o = face_mask_float(H, W, T, ou, ov, scale, host=False)
    m_r = face_mask_float(H, W, T, ru, rv, scale, host=False)
    x = (m_o.to(torch.int32) ^ m_r.to(torch.int32)) & 0xFFF
    fc_t = _popcount12(x & 0x3)
    fc_s = _popcount12(x & 0xFFC)
    f_o = _positive_faces(m_o, H, W, T)
    f_r = _positive_faces(m_r, H, W, T)
    e_o, n_o = trajectory_graph(f_o, H, W, T)
    e_r, n_r = trajectory_graph(f_r, H, W, T)
    iso = f_o == f_r and e_o == e_r
    # field.py:346-372 psnr on the device (float64; the mean's summation
    # order differs from numpy's, so the last bits may)
    lo, hi, _ = device_range(ou, ov)
    rng = hi - lo
    du, dv = ou.double() - ru.double(), ov.double() - rv.double()
    mse = 0.5 * (float((du * du).mean().item()) + float((dv * dv).mean().item()))
    p = math.inf if mse == 0.0 else (-math.inf if rng == 0.0 else
                                     20.0 * math.log10(rng) - 10.0 * math.log10(mse))
    max_err = max(float(du.abs().max().item()), float(dv.abs().max().item()))
    cr = orig.nbytes / archive_size if archive_size else float("nan")
    return VerifyReport(cr=cr, psnr=p, max_abs_err=max_err,
                        fc_t=fc_t, fc_s=fc_s, n_traj_orig=n_o,
                        n_traj_recon=n_r, isomorphic=iso)


# --------------------------------------------------------- residual stats
# tracking.py:199-268: distribution summaries of a symbol stream (0 = escape)
# for `vfcp stats`; the run detection is vectorised (boundaries of the
# center-symbol mask) instead of a Python loop over the stream.

@dataclass
class ResidualStats:
    folded_pmf: np.ndarray        # P(|idx| = m), m = 0.. (escapes excluded)
    tail_ccdf: np.ndarray         # P(|idx| >= m)
    overflow_rate: float
    run_lengths: np.ndarray       # maximal runs of the center symbol
    run_ccdf: np.ndarray          # P(run >= L), L = 1..max
    run_mean: float
    run_percentiles: dict         # {75: ..., 80: ..., 85: ..., 90: ...}

    def write_pmf_csv(self, path) -> None:
        with Path(path).open("w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["magnitude", "pmf", "ccdf"])
            for m, (p, c) in enumerate(zip(self.folded_pmf, self.tail_ccdf)):
                w.writerow([m, f"{p:.10g}", f"{c:.10g}"])

    def write_runs_csv(self, path) -> None:
        with Path(path).open("w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["run_length", "ccdf"])
            for L, c in enumerate(self.run_ccdf, start=1):
                w.writerow([L, f"{c:.10g}"])
            w.writerow([])
            w.writerow(["mean", f"{self.run_mean:.10g}"])
            for q, val in sorted(self.run_percentiles.items()):
                w.writerow([f"p{q}", f"{val:.10g}"])


def residual_stats(symbols, radius: int) -> ResidualStats:
    """tracking.py:228-268."""
    symbols = np.asarray(symbols, dtype=np.int64)
    overflow = symbols == 0
    mags = np.abs(symbols[~overflow] - radius)
    if mags.size:
        pmf = np.bincount(mags) / mags.size
        ccdf = pmf[::-1].cumsum()[::-1]
    else:
        pmf = np.array([0.0])
        ccdf = np.array([0.0])
    c = np.concatenate(([False], symbols == radius, [False])).astype(np.int8)
    d = np.diff(c)
    runs = (np.flatnonzero(d == -1) - np.flatnonzero(d == 1)).astype(np.int64)
    if runs.size:
        rc = np.bincount(runs, minlength=int(runs.max()) + 1)[1:]
        run_ccdf = rc[::-1].cumsum()[::-1] / runs.size
        mean = float(runs.mean())
        pct = {q: float(np.percentile(runs, q)) for q in (75, 80, 85, 90)}
    else:
        run_ccdf = np.array([0.0])
        mean = 0.0
        pct = {q: 0.0 for q in (75, 80, 85, 90)}
    ov_rate = float(overflow.mean()) if symbols.size else 0.0
    return ResidualStats(folded_pmf=pmf, tail_ccdf=ccdf, overflow_rate=ov_rate,
                         run_lengths=runs, run_ccdf=run_ccdf, run_mean=mean,
                         run_percentiles=pct)
