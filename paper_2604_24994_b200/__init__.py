"""paper_2604_24994_b200 -- B200-native Power Foam rasterizer (arXiv 2604.24994).

Thin ctypes binding of the C-ABI library ``libpowerfoam.so`` (include/powerfoam.h).
Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  PyTorch supplies device memory, streams and process groups.
There is no CPU fallback: if the library cannot be loaded, every entry point
raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from . import _build

__all__ = ["PFError", "Renderer", "render", "load_library", "PF_VALIDATE", "PF_STATIC_SCENE",
           "PF_INFERENCE", "STAGES"]

PF_PINHOLE, PF_FISHEYE = 0, 1
PF_VALIDATE = 1
PF_STATIC_SCENE = 2
PF_INFERENCE = 4
STAGES = ["K0_edge_records", "K1_preprocess", "K2_scan", "K3_emit", "K4_sort", "K5_ranges",
          "K6_forward", "K7_backward", "K8_unpack"]
_STATUS = {0: "PF_OK", 1: "PF_ERR_INVALID_ARGUMENT", 2: "PF_ERR_CUDA",
           3: "PF_ERR_OUT_OF_MEMORY", 4: "PF_ERR_STATE"}

EXPORTS = ["pf_create_scene", "pf_render_forward", "pf_render_forward_ex", "pf_render_backward",
           "pf_render_backward_ex", "pf_trace_forward", "pf_destroy",
           "pf_last_error", "pf_debug_binning", "pf_debug_counters", "pf_launch_count",
           "pf_set_profiling", "pf_stage_times", "pf_last_pair_counts",
           "pf_cech_create", "pf_cech_destroy", "pf_cech_last_error", "pf_cech_build",
           "pf_connect_loss", "pf_cech_launch_count"]


class PFError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


class _Camera(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32),
                ("fx", C.c_float), ("fy", C.c_float), ("cx", C.c_float), ("cy", C.c_float),
                ("c2w", C.c_float * 12), ("near_plane", C.c_float), ("model", C.c_int32)]


class _SceneDesc(C.Structure):
    _fields_ = [("num_cells", C.c_int64), ("num_edges", C.c_int64),
                ("sites", C.c_void_p), ("weights", C.c_void_p), ("radii", C.c_void_p),
                ("density", C.c_void_p), ("rgb", C.c_void_p), ("nbr_offsets", C.c_void_p),
                ("nbr_indices", C.c_void_p), ("background", C.c_float * 3),
                ("flags", C.c_uint32), ("normals", C.c_void_p),
                ("num_detail", C.c_int32), ("sv_gamma", C.c_float), ("sv_tau", C.c_float),
                ("sv_axes", C.c_float * 24), ("detail_uv", C.c_void_p),
                ("detail_disp", C.c_void_p), ("detail_sv", C.c_void_p)]


class _Grads(C.Structure):
    _fields_ = [("sites", C.c_void_p), ("weights", C.c_void_p), ("radii", C.c_void_p),
                ("density", C.c_void_p), ("rgb", C.c_void_p), ("normals", C.c_void_p),
                ("detail_uv", C.c_void_p), ("detail_disp", C.c_void_p),
                ("detail_sv", C.c_void_p)]


_lib = None


def load_library(build_if_missing: bool = True):
    """Loads libpowerfoam.so (building it with nvcc if absent or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if os.environ.get("PF_LIBRARY_PATH"):      # A/B variant of the same sources
        path = os.environ["PF_LIBRARY_PATH"]
        build_if_missing = False
    if build_if_missing:
        try:
            path = _build.build()
        except Exception:  # no nvcc on this box: use the shipped .so if present
            if not os.path.exists(path):
                raise
    if not os.path.exists(path):
        raise RuntimeError(f"libpowerfoam.so not found at {path} (run __graft_entry__.build())")
    L = C.CDLL(path)
    P, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.pf_create_scene.argtypes = [C.POINTER(_SceneDesc), C.POINTER(C.c_void_p), P]
    L.pf_render_forward.argtypes = [P, C.POINTER(_Camera), i32, P, P]
    L.pf_render_forward_ex.argtypes = [P, C.POINTER(_Camera), i32, P, P, P]
    L.pf_render_backward.argtypes = [P, C.POINTER(_Camera), i32, P, P, P, P, P, P, P]
    L.pf_render_backward_ex.argtypes = [P, C.POINTER(_Camera), i32, P, C.POINTER(_Grads), P]
    L.pf_trace_forward.argtypes = [P, C.POINTER(_Camera), i32, P, P, P]
    L.pf_destroy.argtypes = [P]
    L.pf_last_error.restype = C.c_char_p
    L.pf_debug_binning.argtypes = [P, C.POINTER(_Camera), P, P, P, P, P, P, C.POINTER(i64), P]
    L.pf_debug_counters.argtypes = [P, C.POINTER(_Camera), P, P]
    L.pf_launch_count.argtypes = [P]
    L.pf_launch_count.restype = i64
    L.pf_set_profiling.argtypes = [P, C.c_int]
    L.pf_stage_times.argtypes = [P, P, P]
    L.pf_last_pair_counts.argtypes = [P, P, i32]
    L.pf_cech_create.argtypes = [C.POINTER(C.c_void_p)]
    L.pf_cech_destroy.argtypes = [P]
    L.pf_cech_last_error.restype = C.c_char_p
    L.pf_cech_build.argtypes = [P, i64, P, P, P, P, i64, C.POINTER(i64), P]
    L.pf_connect_loss.argtypes = [i64, P, P, P, P, P, P, P, P]
    L.pf_cech_launch_count.argtypes = [P]
    L.pf_cech_launch_count.restype = i64
    for name in EXPORTS:
        getattr(L, name).restype = getattr(L, name).restype or C.c_int
    L.pf_last_error.restype = C.c_char_p
    L.pf_cech_last_error.restype = C.c_char_p
    L.pf_launch_count.restype = i64
    L.pf_cech_launch_count.restype = i64
    _lib = L
    return L


def _check(status: int):
    if status != 0:
        raise PFError(status, load_library().pf_last_error().decode())


def _cams(cams) -> tuple:
    if not isinstance(cams, (list, tuple)):
        cams = [cams]
    arr = (_Camera * len(cams))()
    for k, c in enumerate(cams):
        arr[k].width, arr[k].height = int(c.width), int(c.height)
        arr[k].fx, arr[k].fy, arr[k].cx, arr[k].cy = (float(c.fx), float(c.fy), float(c.cx),
                                                      float(c.cy))
        m = [float(v) for v in (c.c2w.tolist() if hasattr(c.c2w, "tolist") else c.c2w)]
        for q in range(12):
            arr[k].c2w[q] = m[q]
        arr[k].near_plane = float(c.near if hasattr(c, "near") else c.near_plane)
        arr[k].model = int(getattr(c, "model", 0))
    return arr, len(cams)


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _dev_f32(t, shape=None, device=None, name="tensor"):
    """Pointer of a contiguous f32 CUDA tensor; checks its shape and (if given) device,
    since the kernels write/read exactly the sizes the handle was created with."""
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float32
            and t.is_contiguous()):
        raise TypeError(f"{name}: expected a contiguous float32 CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: on {t.device}, the scene is on {device}")
    return C.c_void_p(t.data_ptr())


class Renderer:
    """Owns one pf_scene handle over caller tensors (kept referenced here).

    sites f32[N,3], weights f32[N], radii f32[N], density f32[N], rgb f32[N,3],
    nbr_offsets i64[N+1], nbr_indices i32[E]: CUDA tensors on one device.
    normals f32[N,3]: dipoles (NEXT-1).  detail: dict(uv f32[N,K,2], disp f32[N,K],
    sv f32[N,K,8,3], axes (8x3 floats), gamma, tau) -- detail sites (NEXT-2).
    """

    def __init__(self, sites, weights, radii, density, rgb, nbr_offsets, nbr_indices,
                 background=(0.0, 0.0, 0.0), flags: int = 0, num_edges: int | None = None,
                 stream=None, normals=None, detail=None):
        L = load_library()
        self.N = int(sites.shape[0])
        self.device = sites.device
        self.has_normals = normals is not None
        self.detail = detail
        self.K = 0 if detail is None else int(detail["uv"].shape[1])
        self._tensors = (sites, weights, radii, density, rgb, nbr_offsets, nbr_indices, normals)
        N, dev = self.N, self.device
        _dev_f32(sites, (N, 3), dev, "sites")
        _dev_f32(weights, (N,), dev, "weights")
        _dev_f32(radii, (N,), dev, "radii")
        _dev_f32(density, (N,), dev, "density")
        _dev_f32(rgb, (N, 3), dev, "rgb")
        if self.has_normals:
            _dev_f32(normals, (N, 3), dev, "normals")
        if detail is not None:
            K = self.K
            _dev_f32(detail["uv"], (N, K, 2), dev, "detail uv")
            _dev_f32(detail["disp"], (N, K), dev, "detail disp")
            _dev_f32(detail["sv"], (N, K, 8, 3), dev, "detail sv")
        if nbr_offsets.dtype != torch.int64 or nbr_indices.dtype != torch.int32:
            raise TypeError("nbr_offsets must be int64 and nbr_indices int32")
        if not (nbr_offsets.is_cuda and nbr_indices.is_cuda):
            raise TypeError("neighbour lists must be CUDA tensors")
        if nbr_offsets.device != dev or nbr_indices.device != dev:
            raise ValueError("neighbour lists must be on the scene's device")
        if not (nbr_offsets.is_contiguous() and nbr_indices.is_contiguous()):
            raise TypeError("neighbour lists must be contiguous")
        if nbr_offsets.dim() != 1 or nbr_offsets.numel() != N + 1:
            raise ValueError(f"nbr_offsets: expected {N + 1} entries, got "
                             f"{tuple(nbr_offsets.shape)}")
        E = int(nbr_indices.numel()) if num_edges is None else int(num_edges)
        d = _SceneDesc()
        d.num_cells = self.N
        d.num_edges = E
        d.sites, d.weights, d.radii = sites.data_ptr(), weights.data_ptr(), radii.data_ptr()
        d.density, d.rgb = density.data_ptr(), rgb.data_ptr()
        d.nbr_offsets = nbr_offsets.data_ptr()
        d.nbr_indices = nbr_indices.data_ptr() if E > 0 else None
        for c in range(3):
            d.background[c] = float(background[c])
        d.flags = int(flags)
        d.normals = normals.data_ptr() if self.has_normals else None
        if detail is not None:
            d.num_detail = self.K
            d.sv_gamma, d.sv_tau = float(detail["gamma"]), float(detail["tau"])
            ax = [float(v) for v in torch.as_tensor(detail["axes"]).reshape(24).tolist()]
            for q in range(24):
                d.sv_axes[q] = ax[q]
            d.detail_uv = detail["uv"].data_ptr()
            d.detail_disp = detail["disp"].data_ptr()
            d.detail_sv = detail["sv"].data_ptr()
        self.background = tuple(float(b) for b in background)
        self.flags = int(flags)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _check(L.pf_create_scene(C.byref(d), C.byref(h), _stream(stream)))
        self._h = h
        self._L = L

    @classmethod
    def from_scene(cls, sc, device="cuda", flags: int = 0):
        """Uploads a pf_synth.Scene-like object (numpy arrays) and wraps it."""
        dev = torch.device(device)
        t = lambda a, dt: torch.as_tensor(a).to(device=dev, dtype=dt).contiguous()
        nrm = getattr(sc, "normals", None)
        det = getattr(sc, "detail", None)
        detail = None
        if det is not None and nrm is not None:
            detail = dict(uv=t(det.uv, torch.float32), disp=t(det.disp, torch.float32),
                          sv=t(det.sv, torch.float32),
                          axes=[float(v) for v in det.axes.reshape(-1)],
                          gamma=float(det.gamma), tau=float(det.tau))
        return cls(t(sc.sites, torch.float32), t(sc.weights, torch.float32),
                   t(sc.radii, torch.float32), t(sc.density, torch.float32),
                   t(sc.rgb, torch.float32), t(sc.nbr_offsets, torch.int64),
                   t(sc.nbr_indices, torch.int32), background=sc.background, flags=flags,
                   normals=None if nrm is None else t(nrm, torch.float32), detail=detail)

    def sibling(self, flags: int):
        """Another handle on the same tensors (e.g. a PF_INFERENCE renderer)."""
        s, w, r, d, c, o, i, n = self._tensors
        return Renderer(s, w, r, d, c, o, i, background=self.background, flags=flags, normals=n,
                        detail=self.detail)

    @property
    def grad_size(self) -> int:
        """Length of the flat gradient buffer: 9N, 12N with dipole normals, plus 27KN
        with K detail sites (uv 2K, disp K, sv 24K per cell)."""
        return (12 if self.has_normals else 9) * self.N + 27 * self.K * self.N

    @property
    def param_names(self):
        names = ["sites", "weights", "radii", "density", "rgb"]
        if self.has_normals:
            names.append("normals")
        if self.K:
            names += ["detail_uv", "detail_disp", "detail_sv"]
        return names

    def params(self):
        s, w, r, d, c, _, _, n = self._tensors
        p = [s, w, r, d, c]
        if self.has_normals:
            p.append(n)
        if self.K:
            p += [self.detail["uv"], self.detail["disp"], self.detail["sv"]]
        return p

    # -------------------------------------------------------------- hot path
    def forward(self, cams, out=None, stream=None, stats=None):
        """Renders the views into out f32[V,H,W,4].  stats: optional dict with
        f32[N] tensors 'contrib' (+= sum T alpha) and 'normal' (+= sum T alpha
        max(n.d,0)^2, dipole scenes)."""
        arr, V = _cams(cams)
        H, W = arr[0].height, arr[0].width
        if out is None:
            out = torch.empty((V, H, W, 4), device=self.device, dtype=torch.float32)
        _dev_f32(out, (V, H, W, 4), self.device, "out")
        ex = None
        if stats is not None:
            ex = (C.c_void_p * 2)(_dev_f32(stats["contrib"], (self.N,), self.device,
                                           "stats contrib").value,
                                  _dev_f32(stats["normal"], (self.N,), self.device,
                                           "stats normal").value
                                  if stats.get("normal") is not None else None)
        _check(self._L.pf_render_forward_ex(self._h, arr, V, C.c_void_p(out.data_ptr()),
                                            ex, _stream(stream)))
        return out

    def trace(self, cams, out=None, stream=None, stats=False):
        """NEXT-4: renders the views with the adjacency-walk ray tracer into out
        f32[V,H,W,4] (pf_trace_forward).  stats=True also returns a dict (rays,
        visited, located, segments, diverged) -- one stream sync."""
        arr, V = _cams(cams)
        H, W = arr[0].height, arr[0].width
        if out is None:
            out = torch.empty((V, H, W, 4), device=self.device, dtype=torch.float32)
        _dev_f32(out, (V, H, W, 4), self.device, "out")
        st = (C.c_int64 * 5)() if stats else None
        _check(self._L.pf_trace_forward(self._h, arr, V, C.c_void_p(out.data_ptr()), st,
                                        _stream(stream)))
        if not stats:
            return out
        keys = ("rays", "visited", "located", "segments", "diverged")
        return out, {k: int(st[i]) for i, k in enumerate(keys)}

    def backward(self, cams, grad_out, grads=None, stream=None):
        """Accumulates dL/dparams into `grads` (dict or flat f32[grad_size] tensor;
        zeros if None)."""
        arr, V = _cams(cams)
        H, W = arr[0].height, arr[0].width
        _dev_f32(grad_out, (V, H, W, 4), self.device, "grad_out")
        if grads is None:
            grads = torch.zeros(self.grad_size, device=self.device, dtype=torch.float32)
        if isinstance(grads, torch.Tensor):
            _dev_f32(grads, (self.grad_size,), self.device, "flat grads")
            views = self.grad_views(grads)
        else:
            views = grads
        shapes = self.grad_shapes()
        g = _Grads()
        for k in ("sites", "weights", "radii", "density", "rgb"):
            setattr(g, k, _dev_f32(views[k], shapes[k], self.device, f"grads[{k!r}]").value)
        g.normals = (_dev_f32(views["normals"], shapes["normals"], self.device,
                              "grads['normals']").value
                     if self.has_normals and "normals" in views else None)
        for k in ("detail_uv", "detail_disp", "detail_sv"):
            setattr(g, k, _dev_f32(views[k], shapes[k], self.device, f"grads[{k!r}]").value
                    if self.K and k in views else None)
        _check(self._L.pf_render_backward_ex(self._h, arr, V, C.c_void_p(grad_out.data_ptr()),
                                             C.byref(g), _stream(stream)))
        return views

    def grad_shapes(self):
        """Shape of every gradient array the backward writes (param_names order)."""
        N, K = self.N, self.K
        sh = {"sites": (N, 3), "weights": (N,), "radii": (N,), "density": (N,), "rgb": (N, 3)}
        if self.has_normals:
            sh["normals"] = (N, 3)
        if K:
            sh.update(detail_uv=(N, K, 2), detail_disp=(N, K), detail_sv=(N, K, 8, 3))
        return sh

    def grad_views(self, flat):
        """Views of a flat gradient buffer as the parameter arrays (one NCCL buffer)."""
        N = self.N
        out = {"sites": flat[0:3 * N].view(N, 3), "weights": flat[3 * N:4 * N],
               "radii": flat[4 * N:5 * N], "density": flat[5 * N:6 * N],
               "rgb": flat[6 * N:9 * N].view(N, 3)}
        if self.has_normals and flat.numel() >= 12 * N:
            out["normals"] = flat[9 * N:12 * N].view(N, 3)
        K = self.K
        if K and flat.numel() >= self.grad_size:
            o = 12 * N
            out["detail_uv"] = flat[o:o + 2 * K * N].view(N, K, 2)
            o += 2 * K * N
            out["detail_disp"] = flat[o:o + K * N].view(N, K)
            o += K * N
            out["detail_sv"] = flat[o:o + 24 * K * N].view(N, K, 8, 3)
        return out

    # ----------------------------------------------------------- debug / stats
    def debug_binning(self, cam, stream=None):
        arr, _ = _cams(cam)
        N, dev = self.N, self.device
        rect = torch.empty((N, 4), device=dev, dtype=torch.int32)
        count = torch.empty(N, device=dev, dtype=torch.int32)
        kb = torch.empty(N, device=dev, dtype=torch.int32)
        P = C.c_int64()
        _check(self._L.pf_debug_binning(self._h, arr, rect.data_ptr(), count.data_ptr(),
                                        kb.data_ptr(), None, None, None, C.byref(P),
                                        _stream(stream)))
        n = max(int(P.value), 1)
        tx, ty = (arr[0].width + 15) // 16, (arr[0].height + 15) // 16
        keys = torch.empty(n, device=dev, dtype=torch.int64)
        vals = torch.empty(n, device=dev, dtype=torch.int32)
        ranges = torch.empty((tx * ty, 2), device=dev, dtype=torch.int32)
        _check(self._L.pf_debug_binning(self._h, arr, rect.data_ptr(), count.data_ptr(),
                                        kb.data_ptr(), keys.data_ptr(), vals.data_ptr(),
                                        ranges.data_ptr(), C.byref(P), _stream(stream)))
        Pn = int(P.value)
        return dict(rect=rect, count=count, keybits=kb, keys=keys[:Pn], vals=vals[:Pn],
                    ranges=ranges, P=Pn)

    def debug_counters(self, cam, stream=None):
        arr, _ = _cams(cam)
        cnt = torch.zeros((arr[0].height, arr[0].width, 4), device=self.device,
                          dtype=torch.int64)
        _check(self._L.pf_debug_counters(self._h, arr, cnt.data_ptr(), _stream(stream)))
        return cnt

    def launch_count(self) -> int:
        return int(self._L.pf_launch_count(self._h))

    def set_profiling(self, on: bool):
        _check(self._L.pf_set_profiling(self._h, int(bool(on))))

    def stage_times(self):
        ms = (C.c_double * 9)()
        n = (C.c_int64 * 9)()
        _check(self._L.pf_stage_times(self._h, ms, n))
        return {STAGES[k]: (float(ms[k]), int(n[k])) for k in range(9)}

    def pair_counts(self, V: int):
        out = (C.c_int64 * V)()
        _check(self._L.pf_last_pair_counts(self._h, out, V))
        return [int(v) for v in out]

    def close(self):
        if getattr(self, "_h", None):
            self._L.pf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _RenderFn(torch.autograd.Function):
    """Differentiable render: inputs are the renderer's parameter tensors
    (Renderer.params(), in param_names order); the neighbour lists and cameras
    are non-differentiable context."""

    @staticmethod
    def forward(ctx, renderer, cams, *params):
        ctx.renderer, ctx.cams = renderer, cams
        return renderer.forward(cams)

    @staticmethod
    def backward(ctx, grad_out):
        r = ctx.renderer
        g = torch.zeros(r.grad_size, device=r.device, dtype=torch.float32)
        v = r.backward(ctx.cams, grad_out.contiguous(), g)
        return (None, None) + tuple(v[k] for k in r.param_names)


def render(renderer: Renderer, cams):
    """Autograd-aware forward over the renderer's parameter tensors."""
    return _RenderFn.apply(renderer, cams, *renderer.params())


# ---------------------------------------------------------------------------
# NEXT-3: Čech graph builder and L_connect
# ---------------------------------------------------------------------------

def _check_cech(status: int):
    if status != 0:
        raise PFError(status, load_library().pf_cech_last_error().decode())


class CechBuilder:
    """GPU Čech complex (all overlapping sphere pairs) as CSR lists."""

    def __init__(self):
        self._L = load_library()
        h = C.c_void_p()
        _check_cech(self._L.pf_cech_create(C.byref(h)))
        self._h = h
        self._cap = 0

    def build(self, sites, radii, stream=None):
        """sites f32[N,3], radii f32[N] (CUDA) -> (nbr_offsets i64[N+1], nbr_indices i32[E])."""
        _dev_f32(sites)
        _dev_f32(radii)
        N = int(sites.shape[0])
        offs = torch.empty(N + 1, device=sites.device, dtype=torch.int64)
        cap = max(self._cap, 16 * N)
        idx = torch.empty(max(cap, 1), device=sites.device, dtype=torch.int32)
        E = C.c_int64()
        _check_cech(self._L.pf_cech_build(self._h, N, C.c_void_p(sites.data_ptr()),
                                          C.c_void_p(radii.data_ptr()),
                                          C.c_void_p(offs.data_ptr()), C.c_void_p(idx.data_ptr()),
                                          cap, C.byref(E), _stream(stream)))
        if E.value > cap:   # first guess too small: size exactly and rebuild
            cap = int(E.value)
            idx = torch.empty(max(cap, 1), device=sites.device, dtype=torch.int32)
            _check_cech(self._L.pf_cech_build(self._h, N, C.c_void_p(sites.data_ptr()),
                                              C.c_void_p(radii.data_ptr()),
                                              C.c_void_p(offs.data_ptr()),
                                              C.c_void_p(idx.data_ptr()), cap, C.byref(E),
                                              _stream(stream)))
        self._cap = max(self._cap, int(E.value * 1.2))
        return offs, idx[:E.value]

    def launch_count(self) -> int:
        return int(self._L.pf_cech_launch_count(self._h))

    def close(self):
        if getattr(self, "_h", None):
            self._L.pf_cech_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def connect_loss(sites, radii, nbr_offsets, nbr_indices, grads=True, stream=None):
    """L_connect: per-cell loss f32[N] and, if grads, (dL/dsites, dL/dradii)
    of its sum."""
    L = load_library()
    N = int(sites.shape[0])
    loss = torch.empty(N, device=sites.device, dtype=torch.float32)
    gs = torch.zeros_like(sites) if grads else None
    gr = torch.zeros_like(radii) if grads else None
    _check_cech(L.pf_connect_loss(N, C.c_void_p(sites.data_ptr()), C.c_void_p(radii.data_ptr()),
                                  C.c_void_p(nbr_offsets.data_ptr()),
                                  C.c_void_p(nbr_indices.data_ptr()), C.c_void_p(loss.data_ptr()),
                                  C.c_void_p(gs.data_ptr()) if grads else None,
                                  C.c_void_p(gr.data_ptr()) if grads else None, _stream(stream)))
    return loss, gs, gr
