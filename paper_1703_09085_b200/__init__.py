"""paper_1703_09085_b200 -- B200-native accumulated-update H-matrix arithmetic.

Thin Python binding over the C-ABI library libhm (include/hm.h): argument
marshalling only.  Every arithmetic step runs in libhm's sm_100a kernels;
PyTorch supplies device memory (for user panels) and the CUDA stream.  There
is no CPU fallback: importing this package without the built library, or
using it without a CUDA device, raises.

    ctx = Context()                       # device 0, torch's current stream
    G = ctx.build(points, areas, leaf_size=32, eta=2.0, eps=1e-4)
    X, Y, Z = G.clone(), G.clone(), G.clone()
    addmul(1.0, X, Y, Z, eps=1e-4)         # Z <- blocktrunc(Z + X Y)
    d = Z.export()                        # host description (numpy arrays)
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = _lib.load()
    return _LIB


class HMError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{_lib.STATUS.get(status, status)}: {msg}")
        self.status = status


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class Context:
    """hm_ctx bound to a device and a CUDA stream.

    torch_allocator=True routes every device allocation of the library through
    torch's caching allocator (hm_allocator hook: torch.cuda.caching_allocator_alloc
    / _delete on the context's stream), so the library's memory is visible to
    and shared with torch; default: the context's private stream-ordered pool
    (no Python in the allocation path)."""

    def __init__(self, device: int = 0, stream=None, torch_allocator=False):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_1703_09085_b200 needs a CUDA device (B200, sm_100a); no CPU fallback")
        self.device = device
        with torch.cuda.device(device):
            s = stream if stream is not None else torch.cuda.current_stream(device)
        self.stream = s
        self._alloc = None
        if torch_allocator:
            def _a(nbytes, stream_ptr, user):
                try:
                    return torch.cuda.caching_allocator_alloc(int(nbytes), device, s)
                except Exception:
                    return None

            def _f(ptr, nbytes, stream_ptr, user):
                torch.cuda.caching_allocator_delete(int(ptr))

            self._alloc = _lib.Allocator(_lib.ALLOC_FN(_a), _lib.FREE_FN(_f), None)   # kept alive with the context
        h = C.c_void_p()
        st = lib().hm_ctx_create(device, C.c_void_p(s.cuda_stream),
                                 C.byref(self._alloc) if self._alloc is not None else None, C.byref(h))
        if st != 0:
            raise HMError(st, "hm_ctx_create failed")
        self.h = h

    def check(self, st):
        if st != 0:
            raise HMError(st, lib().hm_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            lib().hm_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        self.check(lib().hm_sync(self.h))

    def trim(self):
        """Give back the context's workspaces and cached pool memory (hm_trim)."""
        self.check(lib().hm_trim(self.h))

    # ---- construction
    def build(self, points, areas, leaf_size, eta, eps, kernel=0, normals=None):
        """kernel 0: single layer G, 1: (G+G^T)/2, 2: double layer K + I/2 (needs normals)."""
        pts = np.ascontiguousarray(points, dtype=np.float64)
        ar = np.ascontiguousarray(areas, dtype=np.float64)
        nr = None if normals is None else np.ascontiguousarray(normals, dtype=np.float64)
        n = len(ar)
        perm = np.empty(n, np.int64)
        h = C.c_void_p()
        self.check(lib().hm_build_nrm(self.h, _ptr(pts, C.c_double), _ptr(ar, C.c_double),
                                      _ptr(nr, C.c_double) if nr is not None else None, n, int(kernel),
                                      int(leaf_size), float(eta), float(eps), C.byref(h), _ptr(perm, C.c_int64)))
        m = HMatrix(self, h)
        m.perm = perm
        return m

    def import_desc(self, d):
        keep = {}

        def arr(key, dt):
            a = np.ascontiguousarray(d[key], dtype=dt)
            keep[key] = a
            return a

        hd = _lib.HostDesc()
        hd.n = int(d["n"])
        cs = arr("cl_start", np.int32)
        hd.nclusters = len(cs)
        hd.cl_start = _ptr(cs, C.c_int32)
        for k in ("cl_size", "cl_son0", "cl_nsons", "cl_level"):
            setattr(hd, k, _ptr(arr(k, np.int32), C.c_int32))
        hd.cl_bbox = _ptr(arr("cl_bbox", np.float64), C.c_double)
        br = arr("bl_row", np.int32)
        hd.nblocks = len(br)
        hd.bl_row = _ptr(br, C.c_int32)
        for k in ("bl_col", "bl_kind", "bl_son0", "bl_nsons", "bl_rank"):
            setattr(hd, k, _ptr(arr(k, np.int32), C.c_int32))
        hd.bl_off = _ptr(arr("bl_off", np.int64), C.c_int64)
        f = arr("factors", np.float64)
        hd.factors = _ptr(f, C.c_double)
        hd.nfactors = len(f)
        dn = arr("dense", np.float64)
        hd.dense = _ptr(dn, C.c_double)
        hd.ndense = len(dn)
        if d.get("perm") is not None:
            hd.perm = _ptr(arr("perm", np.int64), C.c_int64)
        h = C.c_void_p()
        self.check(lib().hm_import(self.h, C.byref(hd), C.byref(h)))
        m = HMatrix(self, h)
        m.perm = keep.get("perm")
        return m

    # ---- profiling
    def profile(self, on=True):
        self.check(lib().hm_profile_enable(self.h, 1 if on else 0))

    def profile_reset(self):
        self.check(lib().hm_profile_reset(self.h))

    def profile_get(self):
        p = _lib.Prof()
        self.check(lib().hm_profile_get(self.h, C.byref(p)))
        out = {}
        for i in range(p.count):
            name = bytes(p.name[i]).split(b"\0", 1)[0].decode()
            out[name] = dict(ms=p.ms[i], launches=p.launches[i], flops=p.flops[i], bytes=p.bytes[i])
        return out

    def last_stats(self):
        s = _lib.Stats()
        self.check(lib().hm_stats(self.h, None, C.byref(s)))
        return {k: getattr(s, k) for k, _ in _lib.Stats._fields_}


class HMatrix:
    """Opaque hm_mat owned by its context."""

    def __init__(self, ctx: Context, h):
        self.ctx = ctx
        self.h = h
        self.perm = None

    def free(self):
        if self.h is not None and self.ctx.h is not None:
            self.ctx.check(lib().hm_free(self.ctx.h, self.h))
        self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def clone(self):
        h = C.c_void_p()
        self.ctx.check(lib().hm_clone(self.ctx.h, self.h, C.byref(h)))
        m = HMatrix(self.ctx, h)
        m.perm = self.perm
        return m

    def stats(self):
        s = _lib.Stats()
        self.ctx.check(lib().hm_stats(self.ctx.h, self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in _lib.Stats._fields_}

    def export_sizes(self):
        nf, nd = C.c_int64(), C.c_int64()
        self.ctx.check(lib().hm_export_sizes(self.ctx.h, self.h, C.byref(nf), C.byref(nd)))
        return nf.value, nd.value

    def export(self, pinned=False, bufs=None):
        """Host description (dict of numpy arrays).  The payloads are written by
        the library straight into host arrays (hm_export_into): freshly
        allocated ones (pinned=True: page-locked, full-bandwidth D2H), or the
        caller's preallocated (e.g. pinned) float64 buffers bufs = (factors,
        dense) if they are large enough."""
        import torch
        nf, nd = self.export_sizes()

        def buf(cnt, pre):
            if pre is not None and pre.size >= cnt:
                return pre[:cnt]
            if pinned:
                return torch.empty(max(cnt, 1), dtype=torch.float64, pin_memory=True).numpy()[:cnt]
            return np.empty(cnt, np.float64)

        fbuf = buf(nf, bufs[0] if bufs else None)
        dbuf = buf(nd, bufs[1] if bufs else None)
        nf, nd = C.c_int64(nf), C.c_int64(nd)
        hd = _lib.HostDesc()
        self.ctx.check(lib().hm_export_into(self.ctx.h, self.h, C.byref(hd),
                                            C.c_void_p(fbuf.ctypes.data) if nf.value else None,
                                            C.c_void_p(dbuf.ctypes.data) if nd.value else None))
        nc, nb = hd.nclusters, hd.nblocks

        def cp(p, cnt, dt):
            if not p or cnt == 0:
                return np.zeros(0, dt)
            return np.ctypeslib.as_array(p, shape=(cnt,)).astype(dt, copy=True)

        d = dict(n=np.int64(hd.n))
        for k in ("cl_start", "cl_size", "cl_son0", "cl_nsons", "cl_level"):
            d[k] = cp(getattr(hd, k), nc, np.int32)
        d["cl_bbox"] = cp(hd.cl_bbox, 6 * nc, np.float64).reshape(nc, 6) if hd.cl_bbox else np.zeros((0, 6))
        for k in ("bl_row", "bl_col", "bl_kind", "bl_son0", "bl_nsons", "bl_rank"):
            d[k] = cp(getattr(hd, k), nb, np.int32)
        d["bl_off"] = cp(hd.bl_off, nb, np.int64)
        d["factors"] = fbuf
        d["dense"] = dbuf
        d["perm"] = cp(hd.perm, hd.n, np.int64) if hd.perm else None
        return d


def addmul(alpha, X: HMatrix, Y: HMatrix, Z: HMatrix, eps):
    """Z <- blocktrunc(Z + alpha X Y) (hm_addmul)."""
    Z.ctx.check(lib().hm_addmul(Z.ctx.h, float(alpha), X.h, Y.h, Z.h, float(eps)))


def addmul_std(alpha, X: HMatrix, Y: HMatrix, Z: HMatrix, eps):
    """Standard immediate-update product (hm_addmul_std)."""
    Z.ctx.check(lib().hm_addmul_std(Z.ctx.h, float(alpha), X.h, Y.h, Z.h, float(eps)))


def inv(G: HMatrix, eps):
    """In-place H-inversion with accumulated updates (hm_inv, Fig. 8)."""
    G.ctx.check(lib().hm_inv(G.ctx.h, G.h, float(eps)))


def lr(G: HMatrix, eps):
    """In-place H-LR with accumulated updates (hm_lr): strict lower part = L
    (unit diagonal), upper part = R."""
    G.ctx.check(lib().hm_lr(G.ctx.h, G.h, float(eps)))


def chol(G: HMatrix, eps, shift=0.0):
    """In-place H-Cholesky with accumulated updates of G + shift I (hm_chol);
    lower part = L.  Raises HMError(HM_EPIVOT) naming the cluster on breakdown."""
    G.ctx.check(lib().hm_chol(G.ctx.h, G.h, float(eps), float(shift)))


def matvec(G: HMatrix, x, y, alpha=1.0, beta=0.0, op=0):
    """y <- alpha op(G) x + beta y for torch CUDA float64 tensors (n x c, column-major
    = x.T contiguous, or 1-D)."""
    import torch
    assert x.is_cuda and y.is_cuda and x.dtype == torch.float64 and y.dtype == torch.float64
    n = x.shape[0]
    ncols = 1 if x.dim() == 1 else x.shape[1]
    if x.dim() == 2:
        assert x.stride(0) == 1 and y.stride(0) == 1, "panels must be column-major (stride(0) == 1)"
        ldx, ldy = x.stride(1), y.stride(1)
    else:
        ldx = ldy = n
    G.ctx.check(lib().hm_matvec_thin(G.ctx.h, G.h, int(op), float(alpha), C.c_void_p(x.data_ptr()), ldx,
                                     float(beta), C.c_void_p(y.data_ptr()), ldy, ncols))


SOLVE_OPS = {"L": 0, "R": 1, "LT": 2, "RT": 3, "Lc": 4, "LcT": 5}


def solve(F: HMatrix, x, op):
    """x <- op(F)^{-1} x in place (hm_solve_thin); x: torch CUDA float64 n x c
    column-major (or 1-D); op in 'L', 'R', 'LT', 'RT', 'Lc', 'LcT'."""
    import torch
    assert x.is_cuda and x.dtype == torch.float64
    ncols = 1 if x.dim() == 1 else x.shape[1]
    ldx = x.shape[0] if x.dim() == 1 else x.stride(1)
    if x.dim() == 2:
        assert x.stride(0) == 1, "panels must be column-major (stride(0) == 1)"
    F.ctx.check(lib().hm_solve_thin(F.ctx.h, F.h, SOLVE_OPS[op], C.c_void_p(x.data_ptr()), ldx, ncols))


def precond_error(G: HMatrix, F: HMatrix, kind="lr", iters=30, seed=1703):
    """||I - F^{-1} G||_2 by power iteration (hm_precond_error)."""
    out = C.c_double()
    G.ctx.check(lib().hm_precond_error(G.ctx.h, G.h, F.h, {"lr": 0, "chol": 1, "inv": 2}[kind], int(iters),
                                       C.c_uint64(int(seed)), C.byref(out)))
    return out.value


def test_trunc_batched(ctx: Context, stacks, eps, timed=False):
    """Kernel-level parity export: list of (A (m x l), B (n x l)) numpy arrays ->
    list of (U_k, V_k S_k) numpy arrays, ranks, sigmas (hm_test_trunc_batched);
    timed=True also returns the device ms of the C-ABI call (CUDA events on the
    context stream, after the stacks are uploaded)."""
    import torch
    nj = len(stacks)
    m = np.array([a.shape[0] for a, b in stacks], np.int32)
    n = np.array([b.shape[0] for a, b in stacks], np.int32)
    l = np.array([a.shape[1] for a, b in stacks], np.int32)
    kcap = np.array([max(min(min(mm, ll), min(nn, ll)), 1) for mm, nn, ll in zip(m, n, l)], np.int64)
    a_off = np.zeros(nj, np.int64)
    b_off = np.zeros(nj, np.int64)
    o_off = np.zeros(nj, np.int64)
    p_off = np.zeros(nj, np.int64)
    ta = tb = to = tp = 0
    for i in range(nj):
        a_off[i], b_off[i], o_off[i], p_off[i] = ta, tb, to, tp
        ta += int(m[i]) * int(l[i]) + 1
        tb += int(n[i]) * int(l[i]) + 1
        to += int(m[i]) * int(kcap[i]) + 1
        tp += int(n[i]) * int(kcap[i]) + 1
    dev = torch.device("cuda", ctx.device)
    A = torch.zeros(ta, dtype=torch.float64, device=dev)
    B = torch.zeros(tb, dtype=torch.float64, device=dev)
    UA = torch.zeros(to, dtype=torch.float64, device=dev)
    UB = torch.zeros(tp, dtype=torch.float64, device=dev)
    ha = np.zeros(ta)
    hb = np.zeros(tb)
    for i, (a, b) in enumerate(stacks):
        ha[a_off[i]:a_off[i] + a.size] = np.asarray(a, np.float64).ravel(order="F")
        hb[b_off[i]:b_off[i] + b.size] = np.asarray(b, np.float64).ravel(order="F")
    A.copy_(torch.from_numpy(ha))
    B.copy_(torch.from_numpy(hb))
    torch.cuda.synchronize(dev)
    ranks = np.zeros(nj, np.int32)
    qs = [int(min(mm, nn, ll)) for mm, nn, ll in zip(m, n, l)]
    sig = np.zeros(max(sum(qs), 1))
    if timed:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
    ctx.check(lib().hm_test_trunc_batched(
        ctx.h, nj, _ptr(m, C.c_int32), _ptr(n, C.c_int32), _ptr(l, C.c_int32),
        C.c_void_p(A.data_ptr()), _ptr(a_off, C.c_int64), C.c_void_p(B.data_ptr()), _ptr(b_off, C.c_int64),
        C.c_void_p(UA.data_ptr()), _ptr(o_off, C.c_int64), C.c_void_p(UB.data_ptr()), _ptr(p_off, C.c_int64),
        float(eps), _ptr(ranks, C.c_int32), _ptr(sig, C.c_double)))
    ms = None
    if timed:
        e1.record(ctx.stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1)
    ua = UA.cpu().numpy()
    ub = UB.cpu().numpy()
    out, sigmas, o = [], [], 0
    for i in range(nj):
        k = int(ranks[i])
        U = ua[o_off[i]:o_off[i] + int(m[i]) * k].reshape((int(m[i]), k), order="F")
        V = ub[p_off[i]:p_off[i] + int(n[i]) * k].reshape((int(n[i]), k), order="F")
        out.append((U, V))
        sigmas.append(sig[o:o + qs[i]].copy())
        o += qs[i]
    if timed:
        return out, ranks, sigmas, ms
    return out, ranks, sigmas


def test_eval_batched(H: HMatrix, jobs, split_threshold=0.0):
    """Kernel-level parity export of the A2 step (hm_test_eval_batched):
    jobs = list of (block id, trans, coef, V numpy (rows x w)) -> list of
    out numpy arrays (zero-initialised, out += coef op(H|_b) V)."""
    import torch
    ctx = H.ctx
    dev = torch.device("cuda", ctx.device)
    nj = len(jobs)
    vs, outs = [], []
    blk = np.array([j[0] for j in jobs], np.int32)
    tr = np.array([1 if j[1] else 0 for j in jobs], np.int32)
    coef = np.array([j[2] for j in jobs], np.float64)
    d = H.export()
    cz = d["cl_size"]
    ldv = np.zeros(nj, np.int32)
    ldo = np.zeros(nj, np.int32)
    w = np.zeros(nj, np.int32)
    v_off = np.zeros(nj, np.int64)
    o_off = np.zeros(nj, np.int64)
    tv = to = 0
    for i, (b, t, c, V) in enumerate(jobs):
        rows_out = int(cz[d["bl_col"][b]] if t else cz[d["bl_row"][b]])
        assert V.shape[0] == int(cz[d["bl_row"][b]] if t else cz[d["bl_col"][b]])
        ldv[i], ldo[i], w[i] = V.shape[0], rows_out, V.shape[1]
        v_off[i], o_off[i] = tv, to
        tv += V.size + 1
        to += rows_out * V.shape[1] + 1
    hv = np.zeros(max(tv, 1))
    for i, j in enumerate(jobs):
        hv[v_off[i]:v_off[i] + j[3].size] = np.asarray(j[3], np.float64).ravel(order="F")
    Vd = torch.from_numpy(hv).to(dev)
    Od = torch.zeros(max(to, 1), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    ctx.check(lib().hm_test_eval_batched(ctx.h, H.h, nj, _ptr(blk, C.c_int32), _ptr(tr, C.c_int32),
                                         _ptr(coef, C.c_double), C.c_void_p(Vd.data_ptr()), _ptr(v_off, C.c_int64),
                                         _ptr(ldv, C.c_int32), C.c_void_p(Od.data_ptr()), _ptr(o_off, C.c_int64),
                                         _ptr(ldo, C.c_int32), _ptr(w, C.c_int32), float(split_threshold)))
    ho = Od.cpu().numpy()
    for i in range(nj):
        outs.append(ho[o_off[i]:o_off[i] + int(ldo[i]) * int(w[i])].reshape((int(ldo[i]), int(w[i])), order="F"))
    return outs


def flush_capture(ctx: Context, level_mask):
    """Record the TRUNC batches of the next addmul (hm_flush_capture)."""
    ctx.check(lib().hm_flush_capture(ctx.h, C.c_uint64(int(level_mask))))


def flush_capture_info(ctx: Context):
    """List of per-level dicts (m, n, l, k arrays, has_data) of the capture."""
    nl = C.c_int64()
    ctx.check(lib().hm_flush_capture_info(ctx.h, -1, C.byref(nl), None, None, None, None, None))
    out = []
    for lev in range(nl.value):
        nj = C.c_int64()
        ctx.check(lib().hm_flush_capture_info(ctx.h, lev, C.byref(nj), None, None, None, None, None))
        a = {k: np.zeros(nj.value, np.int32) for k in ("m", "n", "l", "k")}
        hd = C.c_int()
        ctx.check(lib().hm_flush_capture_info(ctx.h, lev, C.byref(nj), _ptr(a["m"], C.c_int32), _ptr(a["n"], C.c_int32),
                                              _ptr(a["l"], C.c_int32), _ptr(a["k"], C.c_int32), C.byref(hd)))
        a["has_data"] = bool(hd.value)
        out.append(a)
    return out


def flush_replay(ctx: Context, level, eps, reps=1):
    """Replay one captured level's TRUNC batch: (mean device ms, rank sum)."""
    ms = C.c_double()
    rs = C.c_int64()
    ctx.check(lib().hm_flush_replay(ctx.h, int(level), float(eps), int(reps), C.byref(ms), C.byref(rs)))
    return ms.value, rs.value


def flush_capture_free(ctx: Context):
    ctx.check(lib().hm_flush_capture_free(ctx.h))


__all__ = ["Context", "HMatrix", "HMError", "addmul", "addmul_std", "inv", "solve", "precond_error", "chol", "lr", "matvec", "lib", "test_trunc_batched",
           "test_eval_batched", "flush_capture", "flush_capture_info", "flush_replay", "flush_capture_free"]
