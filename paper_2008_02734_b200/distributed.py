"""Exact linear-memory DTW across the GPUs of one box.

One process per GPU (torch.distributed; NCCL on the GPU box, gloo in the CPU
tests).  The recursion of divide._solve (divide.py:148-178) runs level by
level on every rank with identical bookkeeping; only the compute is split:

* A recursion level with at least as many internal nodes as ranks hands each
  rank a set of whole nodes, longest-processing-time first by cell count; a
  rank solves its nodes' find_pivot calls in one batched launch
  (lmdtw_pivot_nodes) and the pivots are exchanged (all_gather).
* A level with fewer nodes than ranks (the top of the tree: one node at
  level 0) is split one step further, into the nodes' forward and reverse
  half passes (diagonal.diag_dtw, diagonal.py:172-223).  With at least as
  many half passes as ranks they are assigned longest-first; with fewer, each
  half pass gets a group of ranks and is cut into contiguous strip ranges
  (shards): every shard runs as its own persistent kernel and its first strip
  reads the previous shard's boundary row straight from that rank's GPU
  memory (CUDA IPC handle, NVLink peer access, lmdtw_half_pass_shard) while
  both run.  The owners exchange the three returned diagonals and every
  rank applies the split-point combine of divide.find_pivot
  (divide.py:122-145; lmdtw_pivot_combine) to the same data.
* Leaves (divide.py:153-157) are sharded the same way; their paths are
  exchanged and stitched in the reference's pre-order.

The returned AlignmentResult (path, cost = core.path_cost, cells_processed,
peak_diag_values, peak_table_cells, pivot_trace) is identical to
divide.linmdtw's -- the partition never changes what is computed, only where.
The only data-path exchange is pivots, half-pass diagonals and leaf paths
(O(M + N) per level), moved by ``_exchange``: raw bytes in tensors through
torch.distributed all_gather -- device tensors under NCCL, so diagonals go
GPU to GPU and the split point is reduced on the device
(lmdtw_pivot_combine_device); no pickling.  Features are replicated on every
rank.  ``align_batch_distributed`` shards a batch of independent pairs
(BASELINE cfg4) longest-first with no exchange but the results.

The compute backend is pluggable: ``DeviceEngine`` drives the C ABI on this
rank's GPU.  The CPU tests drive the same driver with a test engine to check
the partition and exchange logic under gloo.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from .core import AlignmentResult, InvalidInputError, as_series, check_cost_kind, precision_dtype
from .divide import LinMdtwConfig, _c_config
from .textbook import tie_codes


def lpt_assign(weights, world):
    """Longest-processing-time assignment: unit q -> rank, deterministic on
    every rank (ties: lower unit index first, then the lowest loaded rank)."""
    load = [0] * world
    owner = [0] * len(weights)
    for q in sorted(range(len(weights)), key=lambda q: (-int(weights[q]), q)):
        r = min(range(world), key=lambda r: (load[r], r))
        owner[q] = r
        load[r] += int(weights[q])
    return owner


def _cells_upto(kstop, M, N):
    return int(_capi.load().lmdtw_cells_upto(int(kstop), int(M), int(N)))


def _peak(kstop, M, N):
    return int(_capi.load().lmdtw_peak_retained_values(int(kstop), int(M), int(N)))


def _kstops(M, N):
    """find_pivot's forward / reverse stopping diagonals (divide.py:112-114)."""
    K = M + N - 1
    kf = (K + 1) // 2
    kb = kf + 1 if K % 2 == 0 else kf
    return kf, kb


def apportion(world, weights):
    """Ranks per unit, proportional to weight, at least one each (len(weights) <= world)."""
    n = len(weights)
    alloc = [1] * n
    for _ in range(world - n):
        q = max(range(n), key=lambda q: (weights[q] / alloc[q], -q))
        alloc[q] += 1
    return alloc


def strip_ranges(kstop, M, N, H, parts):
    """Contiguous strip ranges [lo, hi) of one half pass with about equal cells."""
    rows = min(M, kstop + 1)
    S = (rows + H - 1) // H
    parts = max(1, min(parts, S))
    cells = [_cells_upto(kstop, min(rows, (a + 1) * H), N) - _cells_upto(kstop, a * H, N) for a in range(S)]
    total = sum(cells)
    bounds, acc, k = [0], 0, 1
    for a in range(S):
        acc += cells[a]
        if k < parts and acc * parts >= total * k and S - (a + 1) >= parts - k:
            bounds.append(a + 1)
            k += 1
    while len(bounds) < parts:  # degenerate tails
        bounds.append(bounds[-1])
    bounds.append(S)
    return [(bounds[q], bounds[q + 1]) for q in range(parts)]


def _shard_idx(kstop, M, N, lo, hi, H):
    """Index range [a, b) of each of the last three diagonals owned by rows
    [lo H, hi H) (idx = min(k, M-1) - i, diagonal.py:36-41)."""
    out = []
    for s3 in range(3):
        k = kstop - 2 + s3
        top, ilo = min(k, M - 1), max(0, k - (N - 1))
        r0, r1 = max(lo * H, ilo), min(hi * H - 1, top)
        out.append((top - r1, top - r0 + 1) if r1 >= r0 else (0, 0))
    return out


class DeviceEngine:
    """This rank's compute through the C ABI, features resident on its GPU."""

    def __init__(self, X: np.ndarray, Y: np.ndarray, cfg: LinMdtwConfig, device: int):
        import torch
        self.device = int(device)
        self.cfg = cfg
        self.prec = 32 if precision_dtype(cfg.precision) == np.float32 else 64
        self.Xh = np.ascontiguousarray(X, dtype=np.float32)
        self.Yh = np.ascontiguousarray(Y, dtype=np.float32)
        self.d = self.Xh.shape[1]
        self.Xd = torch.from_numpy(self.Xh).to(f"cuda:{self.device}")
        self.Yd = torch.from_numpy(self.Yh).to(f"cuda:{self.device}")
        self.lib = _capi.load()

    def _xy(self):
        return (C.c_void_p(self.Xd.data_ptr()), self.Xh.shape[0], C.c_void_p(self.Yd.data_ptr()),
                self.Yh.shape[0])

    def pivot_nodes(self, subs):
        """[(i_off, j_off, M, N)] -> [(i, j, k, total)] (sub-block coordinates)."""
        n = len(subs)
        if n == 0:
            return []
        sub = np.ascontiguousarray(np.asarray(subs, np.int64).reshape(n, 4))
        out = np.zeros((n, 5), np.int64)
        tot = np.zeros(n, np.float64)
        X, M, Y, N = self._xy()
        _capi.check(self.lib.lmdtw_pivot_nodes(
            self.device, X, M, Y, N, self.d, n, _capi.ptr(sub), self.prec,
            1 if self.cfg.pivot_tie_rule == "highest" else 0, _capi.MEM_DEVICE, _capi.ptr(out), _capi.ptr(tot)))
        return [(int(out[q, 0]), int(out[q, 1]), int(out[q, 2]), float(tot[q])) for q in range(n)]

    def half_pass(self, sub, reverse):
        """Three D and three C diagonals of one half pass of find_pivot on the
        sub-block (diagonal.diag_dtw): forward to kf, reverse to kb."""
        i_off, j_off, M, N = sub
        kf, kb = _kstops(M, N)
        kstop = kb if reverse else kf
        lens = [int(self.lib.lmdtw_diag_length(kstop - 2 + s, M, N)) for s in range(3)]
        d = [self._dev_empty(L) for L in lens]
        c = [self._dev_empty(L) for L in lens]
        pd = (C.c_void_p * 3)(*[a.data_ptr() for a in d])
        pc = (C.c_void_p * 3)(*[a.data_ptr() for a in c])
        cells = C.c_int64()
        Xs = self.Xd[i_off:i_off + M]
        Ys = self.Yd[j_off:j_off + N]
        # outputs land in device tensors (the library copies with cudaMemcpyDefault)
        _capi.check(self.lib.lmdtw_half_pass(
            self.device, C.c_void_p(Xs.data_ptr()), M, C.c_void_p(Ys.data_ptr()), N, self.d, kstop,
            1 if reverse else 0, self.prec, _capi.MEM_DEVICE, pd, pc, C.byref(cells)))
        return [d[s][:lens[s]] for s in range(3)], [c[s][:lens[s]] for s in range(3)]

    def _dev_empty(self, n):
        import torch
        dt = torch.float32 if self.prec == 32 else torch.float64
        return torch.empty(max(int(n), 1), dtype=dt, device=f"cuda:{self.device}")

    def strip_height(self):
        return int(self.lib.lmdtw_strip_height(self.prec, self.d))

    def half_pass_shard(self, sub, reverse, lo, hi, bnd_local, bnd_prev):
        """Strips [lo, hi) of one half pass (lmdtw_half_pass_shard): returns
        {slot: (first idx, D segment, C segment)} for this shard's rows."""
        i_off, j_off, M, N = sub
        kf, kb = _kstops(M, N)
        kstop = kb if reverse else kf
        lens = [int(self.lib.lmdtw_diag_length(kstop - 2 + s, M, N)) for s in range(3)]
        d = [self._dev_empty(L) for L in lens]
        c = [self._dev_empty(L) for L in lens]
        pd = (C.c_void_p * 3)(*[a.data_ptr() for a in d])
        pc = (C.c_void_p * 3)(*[a.data_ptr() for a in c])
        cells = C.c_int64()
        Xs = self.Xd[i_off:i_off + M]
        Ys = self.Yd[j_off:j_off + N]
        _capi.check(self.lib.lmdtw_half_pass_shard(
            self.device, C.c_void_p(Xs.data_ptr()), M, C.c_void_p(Ys.data_ptr()), N, self.d, kstop,
            1 if reverse else 0, self.prec, _capi.MEM_DEVICE, lo, hi, bnd_local, bnd_prev, pd, pc, C.byref(cells)))
        out = {}
        for s3, (a, b) in enumerate(_shard_idx(kstop, M, N, lo, hi, self.strip_height())):
            if b > a:
                out[s3] = (a, d[s3][a:b].clone(), c[s3][a:b].clone())
        return out

    def handoff_alloc(self, nbytes):
        ptr = C.c_void_p()
        h = (C.c_ubyte * 64)()
        _capi.check(self.lib.lmdtw_ipc_alloc(self.device, int(nbytes), C.byref(ptr), h))
        return ptr, bytes(h)

    def handoff_open(self, handle):
        ptr = C.c_void_p()
        h = (C.c_ubyte * 64).from_buffer_copy(handle)
        _capi.check(self.lib.lmdtw_ipc_open(self.device, h, C.byref(ptr)))
        return ptr

    def handoff_reset(self, ptr, nbytes):
        _capi.check(self.lib.lmdtw_fill_ones(self.device, ptr, int(nbytes)))

    def handoff_close(self, ptr):
        _capi.check(self.lib.lmdtw_ipc_close(self.device, ptr))

    def handoff_free(self, ptr):
        _capi.check(self.lib.lmdtw_ipc_free(self.device, ptr))

    def combine(self, M, N, fwd_d, fwd_c, bwd_d):
        """Split point from the two halves (divide.py:122-145), reduced on this
        rank's GPU by pivot_kernel (lmdtw_pivot_combine_device); the
        diagonals are device tensors after an NCCL exchange (host tensors
        under gloo are staged by the library)."""
        keep = [a.contiguous() for a in list(fwd_d) + list(fwd_c) + list(bwd_d)]
        fd = (C.c_void_p * 3)(*[a.data_ptr() for a in keep[0:3]])
        fc = (C.c_void_p * 3)(*[a.data_ptr() for a in keep[3:6]])
        bd = (C.c_void_p * 3)(*[a.data_ptr() for a in keep[6:9]])
        ijk = np.zeros(3, np.int64)
        tot = C.c_double()
        _capi.check(self.lib.lmdtw_pivot_combine_device(
            self.device, self.prec, M, N, 1 if self.cfg.pivot_tie_rule == "highest" else 0, fd, fc, bd,
            _capi.ptr(ijk), C.byref(tot)))
        return int(ijk[0]), int(ijk[1]), int(ijk[2]), float(tot.value)

    def leaves(self, subs):
        """[(i_off, j_off, M, N)] -> local forward paths (K, 2) int64."""
        n = len(subs)
        if n == 0:
            return []
        sub = np.ascontiguousarray(np.asarray(subs, np.int64).reshape(n, 4))
        cap = int(sum(M + N - 1 for _, _, M, N in subs))
        path = np.zeros((cap, 2), np.int64)
        plen = np.zeros(n, np.int64)
        tie = np.ascontiguousarray(tie_codes(self.cfg.tie_rule), dtype=np.int32)
        X, M, Y, N = self._xy()
        _capi.check(self.lib.lmdtw_leaf_nodes(self.device, X, M, Y, N, self.d, n, _capi.ptr(sub),
                                              _capi.ptr(tie), self.prec, _capi.MEM_DEVICE, _capi.ptr(path),
                                              _capi.ptr(plen)))
        out, w = [], 0
        for q in range(n):
            out.append(path[w:w + int(plen[q])].copy())
            w += int(plen[q])
        return out

    def path_cost(self, path):
        cost = C.c_double()
        p = np.ascontiguousarray(path, np.int64)
        _capi.check(self.lib.lmdtw_path_cost(_capi.ptr(self.Xh), self.Xh.shape[0], _capi.ptr(self.Yh),
                                             self.Yh.shape[0], self.d, _capi.ptr(p), p.shape[0], self.prec,
                                             C.byref(cost)))
        return float(cost.value)


def _comm_device(group):
    """Where exchanged tensors live: this rank's GPU under NCCL, host under gloo."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


_CODES = None


def _exchange(mine, group):
    """All-gather {int key: [1-D arrays]} from every rank without pickling:
    each rank packs its arrays as raw bytes (8-byte aligned) into one uint8
    tensor plus an int64 header (key, count, then dtype code and length per
    array); sizes, headers and payloads go through dist.all_gather on the
    communication device (GPU under NCCL -- diagonals move device to device).
    Returns {key: [tensors on the communication device]} merged over ranks."""
    import torch
    import torch.distributed as dist
    global _CODES
    if _CODES is None:
        _CODES = [torch.float32, torch.float64, torch.int64, torch.uint8]
    dev = _comm_device(group)
    hdr, parts = [], []
    for key in sorted(mine):
        arrs = mine[key]
        hdr += [int(key), len(arrs)]
        for a in arrs:
            t = (a if isinstance(a, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(a))).reshape(-1)
            t = t.to(dev).contiguous()
            hdr += [_CODES.index(t.dtype), t.numel()]
            b = t.view(torch.uint8)
            parts.append(b)
            if b.numel() % 8:
                parts.append(torch.zeros(8 - b.numel() % 8, dtype=torch.uint8, device=dev))
    world = dist.get_world_size(group)
    h = torch.tensor(hdr, dtype=torch.int64, device=dev)
    p = torch.cat(parts) if parts else torch.zeros(0, dtype=torch.uint8, device=dev)
    sz = torch.tensor([h.numel(), p.numel()], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(sz) for _ in range(world)]
    dist.all_gather(sizes, sz, group=group)
    sizes = [tuple(int(v) for v in x.tolist()) for x in sizes]
    hmax = max(1, max(x[0] for x in sizes))
    pmax = max(8, max(x[1] for x in sizes))
    hp = torch.zeros(hmax, dtype=torch.int64, device=dev)
    hp[:h.numel()] = h
    pp = torch.zeros(pmax, dtype=torch.uint8, device=dev)
    pp[:p.numel()] = p
    hs = [torch.empty_like(hp) for _ in range(world)]
    ps = [torch.empty_like(pp) for _ in range(world)]
    dist.all_gather(hs, hp, group=group)
    dist.all_gather(ps, pp, group=group)
    out = {}
    for r in range(world):
        hr = hs[r][:sizes[r][0]].tolist()
        q = o = 0
        while q < len(hr):
            key, n = hr[q], hr[q + 1]
            q += 2
            arrs = []
            for _ in range(n):
                dt, cnt = _CODES[hr[q]], hr[q + 1]
                q += 2
                nb = cnt * torch.empty(0, dtype=dt).element_size()
                arrs.append(ps[r][o:o + nb].view(dt))
                o += nb + (-nb) % 8
            out[key] = arrs
    return out


def _all_ok(ok, group):
    """Every rank learns whether all ranks succeeded (one all_reduce MIN)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([1 if ok else 0], dtype=torch.int64, device=_comm_device(group))
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return bool(t.item())


def _host(a):
    """Tensor or array -> numpy (host)."""
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def _sharded_half_passes(engine, subs, units, weights, rank, world, group):
    """Fewer half passes than ranks: each gets a group of consecutive ranks and
    is cut into strip shards that run concurrently, shard j's first strip
    reading shard j-1's handoff buffer through CUDA IPC.  Returns
    {unit: (d[3], c[3])} with the merged diagonals, on every rank.  A failure
    on any rank is raised on every rank (collectives stay matched)."""
    import torch
    import torch.distributed as dist
    H = engine.strip_height()
    alloc = apportion(world, weights)
    plan, r = {}, 0  # rank -> (unit, shard index, lo, hi)
    shards_of = {}
    for u, g in enumerate(alloc):
        q, rev = units[u]
        _, _, m, n = subs[q]
        kstop = _kstops(m, n)[rev]
        rngs = strip_ranges(kstop, m, n, H, g)
        shards_of[u] = []
        for j in range(g):
            if j < len(rngs) and rngs[j][1] > rngs[j][0]:
                plan[r] = (u, j, rngs[j][0], rngs[j][1])
                shards_of[u].append(r)
            r += 1
    nmax = max(n for _, _, _, n in subs)
    nbytes = int(_capi.load().lmdtw_handoff_words(nmax, engine.prec)) * 8
    ptr, handle = engine.handoff_alloc(nbytes)
    handles = {k: bytes(_host(v[0]).tobytes())
               for k, v in _exchange({rank: [np.frombuffer(handle, np.uint8)]}, group).items()}
    engine.handoff_reset(ptr, nbytes)
    dist.barrier(group)  # every buffer reads tag -1 before any shard runs
    peer, out, err = None, {}, None
    try:
        if rank in plan:
            u, j, lo, hi = plan[rank]
            prev = None
            if j > 0:
                peer = engine.handoff_open(handles[shards_of[u][j - 1]])
                prev = peer
            for s3, (a, sd, sc) in engine.half_pass_shard(subs[units[u][0]], units[u][1], lo, hi, ptr,
                                                           prev).items():
                out[3 * u + s3] = [np.array([a], np.int64), sd, sc]
    except Exception as e:  # noqa: BLE001 -- re-raised below, after the collective
        err = e
    ok = _all_ok(err is None, group)
    parts = _exchange(out, group) if ok else {}
    dist.barrier(group)  # no shard still reads a peer buffer
    if peer is not None:
        engine.handoff_close(peer)
    engine.handoff_free(ptr)
    if not ok:
        raise err if err is not None else RuntimeError("a sharded half pass failed on another rank")
    dev = _comm_device(group)
    dt = torch.float32 if engine.prec == 32 else torch.float64
    got = {}
    for u, (q, rev) in enumerate(units):
        _, _, m, n = subs[q]
        kstop = _kstops(m, n)[rev]
        lens = [int(_capi.load().lmdtw_diag_length(kstop - 2 + s3, m, n)) for s3 in range(3)]
        d = [torch.full((L,), float("nan"), dtype=dt, device=dev) for L in lens]
        c = [torch.full((L,), float("nan"), dtype=dt, device=dev) for L in lens]
        for s3 in range(3):
            if 3 * u + s3 in parts:
                a_t, sd, sc = parts[3 * u + s3]
                a = int(a_t[0])
                d[s3][a:a + sd.numel()] = sd
                c[s3][a:a + sc.numel()] = sc
        got[u] = (d, c)
    return got


def linmdtw_distributed(X, Y, cost: str = "euclidean", config: LinMdtwConfig | None = None, group=None,
                        engine=None, **overrides) -> AlignmentResult:
    """divide.linmdtw (divide.py:181-213) with the recursion's compute spread
    over the ranks of ``group`` (default: the world).  Every rank returns the
    same AlignmentResult."""
    import torch.distributed as dist
    check_cost_kind(cost)
    cfg = config or LinMdtwConfig(**overrides)
    if config is not None and overrides:
        raise InvalidInputError("pass either a config object or keyword overrides, not both")
    Xs, Ys = as_series(X), as_series(Y)
    if Xs.dim != Ys.dim:
        raise InvalidInputError(f"feature dimension mismatch: {Xs.dim} vs {Ys.dim}")
    _c_config(cfg)  # validates the tie rule
    M, N = len(Xs), len(Ys)
    dtype = precision_dtype(cfg.precision)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if engine is None:
        engine = DeviceEngine(Xs.frames, Ys.frames, cfg, _capi.get_device())

    # node: [i_off, j_off, M, N, left, right, pi, pj, k, total, leaf]
    nodes = [[0, 0, M, N, -1, -1, -1, -1, -1, 0.0, -1]]
    level, leaves = [0], []
    cells, peak_diag, peak_table, nlevels = 0, 0, 0, 0
    while level:
        internal = []
        for q in level:
            _, _, m, n = nodes[q][:4]
            if m < cfg.min_dim or n < cfg.min_dim or m + n <= 5:
                nodes[q][10] = len(leaves)
                leaves.append(q)
            else:
                internal.append(q)
        if not internal:
            break
        nlevels += 1
        subs = [tuple(nodes[q][:4]) for q in internal]
        if len(internal) >= world:
            # whole nodes, longest first
            w = [_cells_upto(_kstops(m, n)[0], m, n) + _cells_upto(_kstops(m, n)[1], m, n) for _, _, m, n in subs]
            owner = lpt_assign(w, world)
            mine = [q for q in range(len(subs)) if owner[q] == rank]
            res = engine.pivot_nodes([subs[q] for q in mine])
            got = _exchange({q: [np.array(v[:3], np.int64), np.array([v[3]], np.float64)]
                             for q, v in zip(mine, res)}, group)
            piv = []
            for q in range(len(subs)):
                ijk, tot = _host(got[q][0]), _host(got[q][1])
                piv.append((int(ijk[0]), int(ijk[1]), int(ijk[2]), float(tot[0])))
        else:
            # forward and reverse half passes as separate units
            units = [(q, rev) for q in range(len(subs)) for rev in (0, 1)]
            w = [_cells_upto(_kstops(*subs[q][2:])[rev], *subs[q][2:]) for q, rev in units]
            if len(units) >= world or not hasattr(engine, "half_pass_shard"):
                owner = lpt_assign(w, world)
                mine = [u for u in range(len(units)) if owner[u] == rank]
                res = {}
                for u in mine:
                    d, c = engine.half_pass(subs[units[u][0]], units[u][1])
                    res[u] = list(d) + list(c)
                got = {u: (v[:3], v[3:]) for u, v in _exchange(res, group).items()}
            else:
                got = _sharded_half_passes(engine, subs, units, w, rank, world, group)
            piv = []
            for q in range(len(subs)):
                fd, fc = got[2 * q]
                bd, _ = got[2 * q + 1]
                piv.append(engine.combine(subs[q][2], subs[q][3], fd, fc, bd))
        nxt = []
        for q, (pi, pj, k, tot) in zip(internal, piv):
            i_off, j_off, m, n = nodes[q][:4]
            kf, kb = _kstops(m, n)
            cells += _cells_upto(kf, m, n) + _cells_upto(kb, m, n)
            peak_diag = max(peak_diag, _peak(kf, m, n), _peak(kb, m, n))
            nodes[q][6:10] = [pi, pj, k, tot]
            nodes.append([i_off, j_off, pi + 1, pj + 1, -1, -1, -1, -1, -1, 0.0, -1])
            nodes[q][4] = len(nodes) - 1
            nodes.append([i_off + pi, j_off + pj, m - pi, n - pj, -1, -1, -1, -1, -1, 0.0, -1])
            nodes[q][5] = len(nodes) - 1
            nxt += [nodes[q][4], nodes[q][5]]
        level = nxt

    # leaves, longest first
    lsubs = [tuple(nodes[q][:4]) for q in leaves]
    owner = lpt_assign([m * n for _, _, m, n in lsubs], world)
    mine = [q for q in range(len(lsubs)) if owner[q] == rank]
    got = {q: _host(v[0]).reshape(-1, 2)
           for q, v in _exchange(dict(zip(mine, ([p] for p in engine.leaves([lsubs[q] for q in mine])))),
                                 group).items()}

    # pre-order DFS: pivot trace and leaf sequence (divide.py:160-178)
    trace, seq, stack = [], [], [0]
    while stack:
        q = stack.pop()
        i_off, j_off, m, n, left, right, pi, pj, k, tot, lf = nodes[q]
        if lf >= 0:
            seq.append(lf)
            cells += m * n
            peak_table = max(peak_table, m * n)
            continue
        trace.append({"i": i_off + pi, "j": j_off + pj, "i_off": i_off, "j_off": j_off, "M": m, "N": n,
                      "sub_i": pi, "sub_j": pj, "total_at_pivot": tot, "diagonal_k": k})
        stack += [right, left]
    parts = []
    for s, lf in enumerate(seq):
        i_off, j_off = nodes[leaves[lf]][:2]
        p = got[lf] + np.array([i_off, j_off], np.int64)
        parts.append(p if s == 0 else p[1:])
    path = np.concatenate(parts, axis=0).astype(np.int64)
    return AlignmentResult(
        cost=engine.path_cost(path), path=path, cells_processed=int(cells), cells_budget=2 * M * N,
        precision=str(dtype), algorithm="linmdtw", peak_diag_values=int(peak_diag),
        peak_table_cells=int(peak_table), pivot_trace=tuple(trace))


def align_batch_distributed(pairs, cost: str = "euclidean", config: LinMdtwConfig | None = None, group=None,
                            aligner=None, **overrides) -> list:
    """divide.align_batch over the ranks of ``group`` (BASELINE cfg4 sharded,
    SURVEY.md 8(e) row 1): pairs are independent, so each rank aligns the
    pairs LPT assigns it (longest first by M*N) in one fused batch on its GPU,
    and the results (path, cost, counters, pivot trace) are exchanged so every
    rank returns the full list in input order.  ``aligner(pairs, config)``
    replaces the local compute (default: align_batch on this rank's GPU)."""
    import torch.distributed as dist
    from .divide import align_batch
    check_cost_kind(cost)
    cfg = config or LinMdtwConfig(**overrides)
    if config is not None and overrides:
        raise InvalidInputError("pass either a config object or keyword overrides, not both")
    series = [(as_series(X), as_series(Y)) for X, Y in pairs]
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    owner = lpt_assign([len(X) * len(Y) for X, Y in series], world)
    mine = [q for q in range(len(series)) if owner[q] == rank]
    run = aligner or (lambda ps, c: align_batch(ps, config=c))
    local = run([series[q] for q in mine], cfg) if mine else []
    keys = ("i", "j", "i_off", "j_off", "M", "N", "sub_i", "sub_j", "diagonal_k")
    pack = {}
    for q, r in zip(mine, local):
        tr = np.array([[e[k] for k in keys] for e in r.pivot_trace], np.int64).reshape(-1, len(keys))
        pack[q] = [np.asarray(r.path, np.int64), np.array([r.cost], np.float64),
                   np.array([r.cells_processed, r.cells_budget, r.peak_diag_values, r.peak_table_cells], np.int64),
                   tr, np.array([e["total_at_pivot"] for e in r.pivot_trace], np.float64)]
    got = _exchange(pack, group)
    dtype = precision_dtype(cfg.precision)
    out = []
    for q in range(len(series)):
        path, c, ints, tr, tots = (_host(a) for a in got[q])
        trace = []
        for row, t in zip(tr.reshape(-1, len(keys)), tots):
            e = {k: int(v) for k, v in zip(keys, row)}
            e["total_at_pivot"] = float(t)
            trace.append(e)
        out.append(AlignmentResult(
            cost=float(c[0]), path=path.reshape(-1, 2).copy(), cells_processed=int(ints[0]),
            cells_budget=int(ints[1]), precision=str(dtype), algorithm="linmdtw",
            peak_diag_values=int(ints[2]), peak_table_cells=int(ints[3]),
            pivot_trace=tuple({k: e[k] for k in ("i", "j", "i_off", "j_off", "M", "N", "sub_i", "sub_j",
                                                   "total_at_pivot", "diagonal_k")} for e in trace)))
    return out
