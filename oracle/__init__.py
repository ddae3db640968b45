"""ctypes binding of the CPU oracle (oracle/pf_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg.  The product package
(paper_2604_24994_b200) never imports this module, and this module never
imports the product package.  See pf_oracle.c's header for what each entry
point computes and which passage of PAPER.md / SPEC.md / SURVEY.md it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pf_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

O1, O2, O3 = 1, 2, 3
T_STOP = 1e-4


class OCamera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("c2w", C.c_float * 12), ("near_plane", C.c_float), ("model", C.c_int32)]


class ODetail(C.Structure):
    _fields_ = [("K", C.c_int32), ("uv", C.c_void_p), ("disp", C.c_void_p), ("sv", C.c_void_p),
                ("axes", C.c_float * 24), ("gamma", C.c_float), ("tau", C.c_float)]


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, OpenMP, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64 = C.c_int64
        L.oracle_bin_cells.argtypes = [i64, P, P, P, P, P, P, P]
        L.oracle_emit_sort.argtypes = [i64, P, P, P, C.c_int32, P, P, P, P, P]
        L.oracle_emit_sort.restype = i64
        L.oracle_tile_ranges.argtypes = [i64, P, C.c_int32, P]
        L.oracle_render.argtypes = [C.c_int, i64, P, P, P, P, P, P, P, P, P, P, P, i64, P, P,
                                    P, P, P, P, C.c_int]
        L.oracle_backward.argtypes = [C.c_int, i64, P, P, P, P, P, P, P, P, P, P, P, i64, P, P,
                                      P, P, P, P, P, P, P, P, P, C.c_int]
        L.oracle_cell_stats.argtypes = [C.c_int, i64, P, P, P, P, P, P, P, P, P, P, P, i64, P,
                                         P, P, C.c_int]
        L.oracle_cech_rows.argtypes = [i64, P, P, i64, P, P, P, P, C.c_int]
        L.oracle_connect_loss.argtypes = [i64, P, P, P, P, P, P, P]
        L.oracle_cell_interval.argtypes = [C.c_int, i64, P, P, P, P, P, P, P, i64, P, P,
                                           C.c_double, P, P]
        L.oracle_pixel_segments.argtypes = [C.c_int, i64, P, P, P, P, P, P, P, P, P, P, P,
                                             C.c_int32, C.c_int32, P, i64]
        L.oracle_tangent_frame.argtypes = [P, P]
        L.oracle_soft_voronoi.argtypes = [P, P, C.c_int32, C.c_double, P]
        L.oracle_detail_probe.argtypes = [i64, P, P, P, P, i64, P, P, C.c_double, P]
        L.oracle_pixel_segments.restype = i64
        L.oracle_pixel_ray.argtypes = [P, C.c_int32, C.c_int32, P, P, P]
        L.oracle_composite.argtypes = [i64, P, P, P, P, P]
        L.oracle_composite.restype = i64
        L.oracle_trace.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, P, i64, P, P, P, C.c_int]
        L.oracle_trace_cells.argtypes = [i64, P, P, P, P, P, P, P, C.c_double, P, i64]
        L.oracle_trace_cells.restype = i64
        L.oracle_num_threads.restype = C.c_int
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def make_camera(cam) -> OCamera:
    oc = OCamera()
    oc.width, oc.height = int(cam.width), int(cam.height)
    oc.fx, oc.fy, oc.cx, oc.cy = cam.fx, cam.fy, cam.cx, cam.cy
    for k, v in enumerate(np.asarray(cam.c2w, np.float32).reshape(12)):
        oc.c2w[k] = float(v)
    oc.near_plane = cam.near
    oc.model = int(getattr(cam, "model", 0))
    return oc


class _SceneArrays:
    def __init__(self, sc):
        self.N = sc.num_cells
        self.sites = _c(sc.sites, np.float32)
        self.weights = _c(sc.weights, np.float32)
        self.radii = _c(sc.radii, np.float32)
        self.density = _c(sc.density, np.float32)
        self.rgb = _c(sc.rgb, np.float32)
        self.off = _c(sc.nbr_offsets, np.int64)
        self.idx = _c(sc.nbr_indices, np.int32)
        if self.idx.size == 0:
            self.idx = np.zeros(1, np.int32)
        self.bg = np.asarray(sc.background, np.float32)
        nrm = getattr(sc, "normals", None)
        self.normals = None if nrm is None else _c(nrm, np.float32)
        det = getattr(sc, "detail", None)
        self.det = None
        if det is not None and self.normals is not None:
            self.uv = _c(det.uv, np.float32)
            self.disp = _c(det.disp, np.float32)
            self.sv = _c(det.sv, np.float32)
            d = ODetail()
            d.K = int(self.uv.shape[1])
            d.uv, d.disp, d.sv = _p(self.uv), _p(self.disp), _p(self.sv)
            for k, v in enumerate(np.asarray(det.axes, np.float32).reshape(24)):
                d.axes[k] = float(v)
            d.gamma, d.tau = float(det.gamma), float(det.tau)
            self.det = d

    def detp(self):
        return None if self.det is None else C.cast(C.pointer(self.det), C.c_void_p)

    def args(self):
        return [self.N, _p(self.sites), _p(self.weights), _p(self.radii), _p(self.density),
                _p(self.rgb), _p(self.off), _p(self.idx), _p(self.bg), _p(self.normals),
                self.detp()]


# ---------------------------------------------------------------------------
# binning specification (fp32)
# ---------------------------------------------------------------------------

def bin_cells(sc, cam):
    """-> rect i32[N,4] (tx0,ty0,tx1,ty1), count i32[N], keybits u32[N]."""
    A = _SceneArrays(sc)
    rect = np.zeros((A.N, 4), np.int32)
    count = np.zeros(A.N, np.int32)
    kb = np.zeros(A.N, np.uint32)
    oc = make_camera(cam)
    lib().oracle_bin_cells(A.N, _p(A.sites), _p(A.weights), _p(A.radii), C.byref(oc),
                           _p(rect), _p(count), _p(kb))
    return rect, count, kb


def binning(sc, cam):
    """Full binning spec: dict(rect, count, keybits, keys u64[P], vals u32[P], ranges u32[T,2])."""
    rect, count, kb = bin_cells(sc, cam)
    tiles_x = (cam.width + 15) // 16
    tiles_y = (cam.height + 15) // 16
    L = lib()
    A = _SceneArrays(sc)
    oc = make_camera(cam)
    P = L.oracle_emit_sort(sc.num_cells, _p(rect), _p(count), _p(kb), tiles_x, None, None,
                           C.byref(oc), _p(A.sites), _p(A.radii))
    keys = np.zeros(max(P, 1), np.uint64)
    vals = np.zeros(max(P, 1), np.uint32)
    L.oracle_emit_sort(sc.num_cells, _p(rect), _p(count), _p(kb), tiles_x, _p(keys), _p(vals),
                       C.byref(oc), _p(A.sites), _p(A.radii))
    ranges = np.zeros((tiles_x * tiles_y, 2), np.uint32)
    L.oracle_tile_ranges(P, _p(keys), tiles_x * tiles_y, _p(ranges))
    return dict(rect=rect, count=count, keybits=kb, keys=keys[:P], vals=vals[:P],
                ranges=ranges, P=int(P), tiles_x=tiles_x, tiles_y=tiles_y)


# ---------------------------------------------------------------------------
# render / backward
# ---------------------------------------------------------------------------

def render(sc, cam, mode=O3, pixels=None, counters=False, signature=False, nthreads=0):
    """Render (double).  pixels: None (full image) or int array [n,2] of (x,y).
    Returns dict(out f64[n,4] or [H,W,4], counters i64[n,4], sig u64[n], nseg, viol)."""
    A = _SceneArrays(sc)
    oc = make_camera(cam)
    if pixels is None:
        n = cam.width * cam.height
        pix = None
    else:
        pix = _c(np.asarray(pixels).reshape(-1, 2), np.int32)
        n = pix.shape[0]
    out = np.zeros((n, 4), np.float64)
    cnt = np.zeros((n, 4), np.int64) if counters else None
    sig = np.zeros(n, np.uint64) if signature else None
    nseg = np.zeros(n, np.int64)
    viol = np.zeros(1, np.int64)
    lib().oracle_render(mode, *A.args(), C.byref(oc), n, _p(pix), _p(out), _p(cnt), _p(sig),
                        _p(nseg), _p(viol), nthreads)
    if pixels is None:
        out = out.reshape(cam.height, cam.width, 4)
    return dict(out=out, counters=cnt, sig=sig, nseg=nseg, viol=int(viol[0]))


def backward(sc, cam, grad_out, mode=O3, pixels=None, nthreads=0):
    """Gradients of L = sum <grad_out, out>.  grad_out f32[H,W,4] (pixels=None) or [n,4].
    Returns dict(sites f64[N,3], weights, radii, density f64[N], rgb f64[N,3])."""
    A = _SceneArrays(sc)
    oc = make_camera(cam)
    if pixels is None:
        n = cam.width * cam.height
        pix = None
    else:
        pix = _c(np.asarray(pixels).reshape(-1, 2), np.int32)
        n = pix.shape[0]
    g = _c(np.asarray(grad_out).reshape(n, 4), np.float32)
    N = A.N
    gs = np.zeros((N, 3)); gw = np.zeros(N); gr = np.zeros(N); gsig = np.zeros(N)
    grgb = np.zeros((N, 3))
    gn = np.zeros((N, 3)) if A.normals is not None else None
    guv = gdisp = gsv = None
    if A.det is not None:
        guv = np.zeros(A.uv.shape); gdisp = np.zeros(A.disp.shape); gsv = np.zeros(A.sv.shape)
    lib().oracle_backward(mode, *A.args(), C.byref(oc), n, _p(pix), _p(g), _p(gs), _p(gw),
                          _p(gr), _p(gsig), _p(grgb), _p(gn), _p(guv), _p(gdisp), _p(gsv),
                          nthreads)
    out = dict(sites=gs, weights=gw, radii=gr, density=gsig, rgb=grgb)
    if gn is not None:
        out["normals"] = gn
    if guv is not None:
        out.update(detail_uv=guv, detail_disp=gdisp, detail_sv=gsv)
    return out


def cell_stats(sc, cam, mode=O3, pixels=None, nthreads=0):
    """Per-cell forward by-products: contrib = sum T_k alpha_k (L_sparse / pruning),
    normal = sum T_k alpha_k max(n.d, 0)^2 (L_normal; dipole scenes only)."""
    A = _SceneArrays(sc)
    oc = make_camera(cam)
    if pixels is None:
        n = cam.width * cam.height
        pix = None
    else:
        pix = _c(np.asarray(pixels).reshape(-1, 2), np.int32)
        n = pix.shape[0]
    contrib = np.zeros(A.N)
    normal = np.zeros(A.N) if A.normals is not None else None
    lib().oracle_cell_stats(mode, *A.args(), C.byref(oc), n, _p(pix), _p(contrib), _p(normal),
                            nthreads)
    return dict(contrib=contrib, normal=normal)


def cell_interval(sc, i, Q, d, t_near=0.0, mode=O2):
    """(hit, t_in, t_out, kinds[kin,kout,jin,jout]) of cell i on the ray Q + t d."""
    A = _SceneArrays(sc)
    Qa = _c(Q, np.float64)
    da = _c(d, np.float64)
    res = np.zeros(2)
    kinds = np.zeros(4, np.int32)
    hit = lib().oracle_cell_interval(mode, A.N, _p(A.sites), _p(A.weights), _p(A.radii),
                                     _p(A.off), _p(A.idx), _p(A.normals), A.detp(), int(i),
                                     _p(Qa), _p(da),
                                     float(t_near), _p(res), _p(kinds))
    return bool(hit), float(res[0]), float(res[1]), kinds


def pixel_segments(sc, cam, x, y, mode=O3, cap=4096):
    """Composited segments of pixel (x,y): list of dicts (cell, t_in, t_out, kin, kout,
    jin, jout, list_pos); kinds 0 sphere, 1 near, 2 plane, 3 dipole."""
    A = _SceneArrays(sc)
    oc = make_camera(cam)
    buf = np.zeros((cap, 8))
    n = lib().oracle_pixel_segments(mode, *A.args(), C.byref(oc), int(x), int(y), _p(buf), cap)
    keys = ("cell", "t_in", "t_out", "kin", "kout", "jin", "jout", "list_pos")
    return [dict(zip(keys, row)) for row in buf[:n]]


def tangent_frame(n):
    """(u, v, m) of a face normal and the chosen axis."""
    nn = _c(n, np.float32)
    out = np.zeros(9)
    k = lib().oracle_tangent_frame(_p(nn), _p(out))
    return out[:3], out[3:6], out[6:], int(k)


def soft_voronoi(q, uv, tau):
    """Soft-Voronoi weights of the chart point q against sites uv [K,2]."""
    qa = _c(q, np.float64); u = _c(uv, np.float32).reshape(-1, 2)
    w = np.zeros(u.shape[0])
    assert lib().oracle_soft_voronoi(_p(qa), _p(u), u.shape[0], float(tau), _p(w)) == 0
    return w


def detail_probe(sc, i, Q, d, t_entry=0.0):
    """Detail evaluation of cell i on the ray Q + t d: dict(parallel, tb, dr, delta, ts,
    col[3], qb[2], qs[2])."""
    A = _SceneArrays(sc)
    Qa = _c(Q, np.float64); da = _c(d, np.float64)
    out = np.zeros(12)
    assert lib().oracle_detail_probe(A.N, _p(A.sites), _p(A.radii), _p(A.normals), A.detp(),
                                     int(i), _p(Qa), _p(da), float(t_entry), _p(out)) == 0
    return dict(parallel=bool(out[0]), tb=out[1], dr=out[2], delta=out[3], ts=out[4],
                col=out[5:8].copy(), qb=out[8:10].copy(), qs=out[10:12].copy())


def pixel_ray(cam, x, y):
    oc = make_camera(cam)
    Q = np.zeros(3); d = np.zeros(3); tn = np.zeros(1)
    lib().oracle_pixel_ray(C.byref(oc), int(x), int(y), _p(Q), _p(d), _p(tn))
    return Q, d, float(tn[0])


def composite(sigma, dt, rgb, bg=(0.0, 0.0, 0.0)):
    sigma = _c(sigma, np.float64); dt = _c(dt, np.float64)
    rgb = _c(np.asarray(rgb).reshape(-1, 3), np.float64)
    bga = _c(bg, np.float64)
    out = np.zeros(4)
    K = lib().oracle_composite(len(sigma), _p(sigma), _p(dt), _p(rgb), _p(bga), _p(out))
    return out, int(K)


def trace(sc, cam, pixels=None, nthreads=0):
    """NEXT-4 adjacency-walk ray tracer (double): dict(out f64[n,4] or [H,W,4],
    stats i64[n,3] = (cells visited, locate calls, composited segments))."""
    A = _SceneArrays(sc)
    oc = make_camera(cam)
    if pixels is None:
        n = cam.width * cam.height
        pix = None
    else:
        pix = _c(np.asarray(pixels).reshape(-1, 2), np.int32)
        n = pix.shape[0]
    out = np.zeros((n, 4), np.float64)
    st = np.zeros((n, 3), np.int64)
    lib().oracle_trace(*A.args(), C.byref(oc), n, _p(pix), _p(out), _p(st), nthreads)
    if pixels is None:
        out = out.reshape(cam.height, cam.width, 4)
        st = st.reshape(cam.height, cam.width, 3)
    return dict(out=out, stats=st)


def trace_cells(sc, Q, d, t_near=0.0, cap=4096):
    """The cells the tracer's walk visits along the ray Q + t d, in order."""
    A = _SceneArrays(sc)
    Qa = _c(Q, np.float64)
    da = _c(d, np.float64)
    cells = np.zeros(cap, np.int32)
    n = lib().oracle_trace_cells(A.N, _p(A.sites), _p(A.weights), _p(A.radii), _p(A.off),
                                 _p(A.idx), _p(Qa), _p(da), float(t_near), _p(cells), cap)
    return [int(c) for c in cells[:min(n, cap)]]


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ---------------------------------------------------------------------------
# NEXT-3: Čech graph and L_connect
# ---------------------------------------------------------------------------

def cech_rows(sites, radii, rows=None, nthreads=0):
    """Brute-force Čech neighbour rows (ascending j).  rows=None -> all cells.
    Returns (offsets i64[n+1], indices i32[E])."""
    sites = _c(sites, np.float32).reshape(-1, 3)
    radii = _c(radii, np.float32).reshape(-1)
    N = sites.shape[0]
    rws = np.arange(N, dtype=np.int64) if rows is None else _c(rows, np.int64)
    n = rws.shape[0]
    counts = np.zeros(n, np.int64)
    L = lib()
    L.oracle_cech_rows(N, _p(sites), _p(radii), n, _p(rws), _p(counts), None, None, nthreads)
    offs = np.zeros(n + 1, np.int64)
    np.cumsum(counts, out=offs[1:])
    idx = np.zeros(max(int(offs[-1]), 1), np.int32)
    L.oracle_cech_rows(N, _p(sites), _p(radii), n, _p(rws), _p(counts), _p(offs[:-1].copy()),
                       _p(idx), nthreads)
    return offs, idx[:int(offs[-1])]


def connect_loss(sites, radii, offsets, indices):
    """L_connect per cell and the gradient of its sum."""
    sites = _c(sites, np.float32).reshape(-1, 3)
    radii = _c(radii, np.float32).reshape(-1)
    N = sites.shape[0]
    off = _c(offsets, np.int64)
    idx = _c(indices, np.int32) if len(indices) else np.zeros(1, np.int32)
    loss = np.zeros(N); gs = np.zeros((N, 3)); gr = np.zeros(N)
    lib().oracle_connect_loss(N, _p(sites), _p(radii), _p(off), _p(idx), _p(loss), _p(gs), _p(gr))
    return dict(loss=loss, sites=gs, radii=gr)
