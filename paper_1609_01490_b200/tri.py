"""Thin ctypes binding of libtri.so (include/tri.h) -- argument marshalling only.

Every function here has the C name and forwards to the library; tensors are
passed as raw device pointers (``tensor.data_ptr()``) with their byte
capacity, and the stream defaults to torch's current CUDA stream.  There is no
compute in Python and no CPU fallback: if libtri.so cannot be loaded the first
call raises.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtri.so")

TRI_OK, TRI_EINVAL, TRI_ERANGE, TRI_ECUDA, TRI_ENOTSUP = 0, -1, -2, -3, -4
TRI_LAMBDA, TRI_BB, TRI_LAMBDA_PERSIST = 0, 1, 2
TRI_LAMBDA_CLC = 7                                           # persistent CTAs, cluster launch control
TRI_DUMMY_FIXED, TRI_DUMMY_PACKED, TRI_DUMMY_DIGEST, TRI_DUMMY_COUNT = 0, 1, 2, 3
TRI_LAMBDA_X, TRI_LAMBDA_N, TRI_LAMBDA_R = 3, 4, 5          # tri_dummy only (section 4.1 variants)
TRI_SQRT_X, TRI_SQRT_N, TRI_SQRT_R = 1, 2, 3
STRATEGIES = {"lambda": TRI_LAMBDA, "bb": TRI_BB, "persist": TRI_LAMBDA_PERSIST,
              "lambda_x": TRI_LAMBDA_X, "lambda_n": TRI_LAMBDA_N, "lambda_r": TRI_LAMBDA_R, "rb": 6,
              "clc": TRI_LAMBDA_CLC, "tc": 8, "bb_tc": 9}
TRI_RB = 6                                                   # tri_dummy / tri_edm, single rank

c_u64, c_i64, c_i32, c_u32, c_vp = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32, ctypes.c_void_p
c_sz = ctypes.c_size_t


class TriMap(ctypes.Structure):
    """tri_map_t (include/tri.h)."""
    _fields_ = [("n", c_i64), ("rho", c_i32), ("diag", c_i32), ("rank", c_i32), ("world", c_i32),
                ("m", c_i64), ("blocks", c_u64), ("cells", c_u64),
                ("omega_begin", c_u64), ("omega_end", c_u64),
                ("row_begin", c_i64), ("row_end", c_i64),
                ("out_offset", c_u64), ("out_cells", c_u64),
                ("waste_lambda", c_u64), ("waste_bb", c_u64),
                ("snap", c_i32), ("reserved", c_i32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


class TetMap(ctypes.Structure):
    """tet_map_t (include/tri.h)."""
    _fields_ = [("n", c_i64), ("rho", c_i32), ("rank", c_i32), ("world", c_i32), ("reserved", c_i32),
                ("m", c_i64), ("blocks", c_u64), ("omega_begin", c_u64), ("omega_end", c_u64),
                ("waste_tet", c_u64), ("waste_bb", c_u64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


class TriError(RuntimeError):
    def __init__(self, code, what):
        self.code = code
        super().__init__(f"{what}: {status_str(code)} ({code})")


_lib = None

SIGNATURES = {
    "tri_map_init": ([ctypes.POINTER(TriMap), c_i64, c_i32, c_i32, c_i32, c_i32, c_i32], c_i32),
    "tri_lambda": ([c_u64, ctypes.POINTER(c_u32), ctypes.POINTER(c_u32)], c_i32),
    "tri_lambda_nodiag": ([c_u64, ctypes.POINTER(c_u32), ctypes.POINTER(c_u32)], c_i32),
    "tri_collide1d": ([ctypes.POINTER(TriMap), c_i32, c_vp, ctypes.c_size_t, c_vp, ctypes.c_size_t, c_vp], c_i32),
    "tri_map_eval": ([c_u64, c_u64, c_vp, c_vp, c_vp], c_i32),
    "tri_map_eval_variant": ([c_i32, c_u64, c_u64, c_vp, c_vp, c_vp], c_i32),
    "tri_map_rows_variant": ([c_i32, c_u64, c_u64, c_vp, c_sz, c_vp], c_i32),
    "tri_dummy": ([ctypes.POINTER(TriMap), c_i32, c_i32, c_vp, ctypes.c_size_t, c_vp], c_i32),
    "tri_edm": ([ctypes.POINTER(TriMap), c_i32, c_vp, c_i32, c_i64, c_sz, c_vp, c_sz, c_vp], c_i32),
    "tri_edm_host": ([ctypes.POINTER(TriMap), c_i32, c_vp, c_i32, c_i64, c_sz, c_vp, c_sz, c_vp, c_sz,
                      c_vp, c_sz, c_u64], c_i32),
    "tri_collide": ([ctypes.POINTER(TriMap), c_i32, c_vp, c_sz, c_vp, c_sz, c_vp, c_sz, c_vp], c_i32),
    "tri_collide_workspace_size": ([ctypes.POINTER(TriMap), c_i32], c_sz),
    "tri_tc_tf32_probe": ([c_vp, c_vp, c_vp, c_vp], c_i32),
    "tri_tc_f16_probe": ([c_vp, c_vp, c_vp, c_vp], c_i32),
    "tri_ca_workspace_size": ([ctypes.POINTER(TriMap)], c_sz),
    "tri_ca_step": ([ctypes.POINTER(TriMap), c_i32, c_vp, c_sz, c_vp, c_sz, c_vp, c_sz, c_vp, c_sz, c_vp, c_vp],
                    c_i32),
    "tri_ca_steps": ([ctypes.POINTER(TriMap), c_i32, c_i32, c_vp, c_sz, c_vp, c_sz, c_vp, c_sz, c_vp, c_sz,
                      c_vp, c_vp], c_i32),
    "tri_ca_run_workspace_size": ([ctypes.POINTER(TriMap)], c_sz),
    "tri_ca_run": ([ctypes.POINTER(TriMap), c_i32, c_i64, c_vp, c_sz, c_vp, c_sz, c_vp, c_sz, c_vp], c_i32),
    "tri_ca_steps_p2p": ([ctypes.POINTER(TriMap), c_i32, c_i32, c_vp, c_sz, c_vp, c_sz, c_vp, c_sz, c_vp, c_sz,
                          c_vp, c_vp, c_vp, c_vp], c_i32),
    "tri_ipc_handle": ([c_vp, c_vp, ctypes.POINTER(c_u64)], c_i32),
    "tri_ipc_open": ([c_vp, c_u64, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp)], c_i32),
    "tri_ipc_close": ([c_vp], c_i32),
    "tet_map_init": ([ctypes.POINTER(TetMap), c_i64, c_i32, c_i32, c_i32], c_i32),
    "tet_lambda": ([c_u64, ctypes.POINTER(c_u32), ctypes.POINTER(c_u32), ctypes.POINTER(c_u32)], c_i32),
    "tet_map_eval": ([c_u64, c_u64, c_vp, c_vp, c_vp], c_i32),
    "tet_lut_bytes": ([c_u32, c_i32], ctypes.c_size_t),
    "tet_lut_build": ([c_u32, c_i32, c_vp, ctypes.c_size_t, c_vp], c_i32),
    "tet_map_eval_lut": ([c_u64, c_u64, c_u32, c_i32, c_vp, c_vp, c_vp, c_vp], c_i32),
    "tet_triplet": ([ctypes.POINTER(TetMap), c_i32, c_vp, c_sz, ctypes.c_double, c_vp, c_sz, c_vp], c_i32),
    "tri_last_launch_count": ([], c_i32),
    "tri_status_str": ([c_i32], ctypes.c_char_p),
}


def lib():
    """Load libtri.so (raises if it is missing -- there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libtri.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        for name, (argt, rest) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = argt
            fn.restype = rest
        _lib = L
    return _lib


def status_str(code: int) -> str:
    return lib().tri_status_str(code).decode()


def _ok(code, what):
    if code != TRI_OK:
        raise TriError(code, what)


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _nbytes(t):
    return 0 if t is None else t.numel() * t.element_size()


def _cap(t):
    """Bytes from t's first element to the end of its storage (a strided view's capacity)."""
    return t.untyped_storage().nbytes() - t.storage_offset() * t.element_size()


def _need(cond, what):
    """Marshalling guard: a tensor of the wrong kind is a caller error, caught before the
    C call (the library checks sizes again, but cannot see dtypes or devices)."""
    if not cond:
        raise TypeError(what)


def _strategy(s):
    return STRATEGIES[s] if isinstance(s, str) else int(s)


# ----------------------------------------------------------------------------- map
def tri_map_init(n, rho, diag=1, rank=0, world=1, snap_rows=1) -> TriMap:
    m = TriMap()
    _ok(lib().tri_map_init(ctypes.byref(m), n, rho, diag, rank, world, snap_rows), "tri_map_init")
    return m


def tri_lambda(omega):
    bi, bj = c_u32(), c_u32()
    _ok(lib().tri_lambda(omega, ctypes.byref(bi), ctypes.byref(bj)), "tri_lambda")
    return bi.value, bj.value


def tri_lambda_nodiag(omega):
    i, j = c_u32(), c_u32()
    _ok(lib().tri_lambda_nodiag(omega, ctypes.byref(i), ctypes.byref(j)), "tri_lambda_nodiag")
    return i.value, j.value


def tri_collide1d(m: TriMap, strategy, intervals, count, stream=None):
    """intervals: (n, 2) float32 CUDA tensor (c, r); count: 8-byte integer CUDA tensor."""
    _need(intervals.is_cuda and intervals.dtype.itemsize == 4 and intervals.is_floating_point()
          and intervals.dim() == 2 and intervals.shape[1] == 2 and intervals.is_contiguous(),
          "tri_collide1d: intervals must be a contiguous (n, 2) float32 CUDA tensor")
    _need(count.is_cuda and count.element_size() == 8 and not count.is_floating_point(),
          "tri_collide1d: count must be an 8-byte integer CUDA tensor")
    _ok(lib().tri_collide1d(ctypes.byref(m), _strategy(strategy), _ptr(intervals), _nbytes(intervals),
                            _ptr(count), _nbytes(count), _stream(stream)), "tri_collide1d")


def tri_map_eval(omega0, count, d_ij, d_fail, stream=None):
    _ok(lib().tri_map_eval(omega0, count, _ptr(d_ij), _ptr(d_fail), _stream(stream)), "tri_map_eval")


def tri_map_rows_variant(variant, omega0, count, d_rows, stream=None):
    """d_rows: int32/uint32 CUDA tensor >= count: the uncorrected variant's row per omega."""
    _need(d_rows.is_cuda and d_rows.element_size() == 4, "tri_map_rows_variant: d_rows must be 4-byte CUDA")
    _ok(lib().tri_map_rows_variant(variant, omega0, count, _ptr(d_rows), _nbytes(d_rows), _stream(stream)),
        "tri_map_rows_variant")


def tri_map_eval_variant(variant, omega0, count, d_fail, d_first, stream=None):
    """Validity scan of a section-4.1 sqrt variant (TRI_SQRT_X / _N / _R)."""
    _ok(lib().tri_map_eval_variant(variant, omega0, count, _ptr(d_fail), _ptr(d_first), _stream(stream)),
        "tri_map_eval_variant")


def tet_map_init(n, rho, rank=0, world=1) -> TetMap:
    m = TetMap()
    _ok(lib().tet_map_init(ctypes.byref(m), n, rho, rank, world), "tet_map_init")
    return m


def tet_lambda(omega):
    i, j, k = c_u32(), c_u32(), c_u32()
    _ok(lib().tet_lambda(omega, ctypes.byref(i), ctypes.byref(j), ctypes.byref(k)), "tet_lambda")
    return i.value, j.value, k.value


def tet_map_eval(omega0, count, d_ijk, d_fail, stream=None):
    _ok(lib().tet_map_eval(omega0, count, _ptr(d_ijk), _ptr(d_fail), _stream(stream)), "tet_map_eval")


def tet_lut_bytes(kmax, shift):
    """Bytes of the succinct layer table (0 on bad arguments); host-only arithmetic."""
    return int(lib().tet_lut_bytes(kmax, shift))


def tet_lut_build(kmax, shift, d_lut, stream=None):
    nb = _nbytes(d_lut) if d_lut is not None else 0
    _ok(lib().tet_lut_build(kmax, shift, _ptr(d_lut), nb, _stream(stream)), "tet_lut_build")


def tet_map_eval_lut(omega0, count, kmax, shift, d_lut, d_ijk, d_fail, stream=None):
    _ok(lib().tet_map_eval_lut(omega0, count, kmax, shift, _ptr(d_lut), _ptr(d_ijk), _ptr(d_fail),
                               _stream(stream)), "tet_map_eval_lut")


# ----------------------------------------------------------------------------- kernels
def tri_dummy(m: TriMap, strategy, mode, out, stream=None):
    _ok(lib().tri_dummy(ctypes.byref(m), _strategy(strategy), mode, _ptr(out), _nbytes(out), _stream(stream)),
        "tri_dummy")


def tri_edm(m: TriMap, strategy, pts, out, stream=None):
    """pts: (n, dim) float32 CUDA tensor (row stride = pts.stride(0)); out: float32 >= out_cells."""
    _need(pts.is_cuda and pts.dtype.itemsize == 4 and pts.is_floating_point() and pts.dim() == 2
          and pts.stride(1) == 1, "tri_edm: pts must be an (n, dim) float32 CUDA tensor, unit column stride")
    _need(out.is_cuda and out.dtype.itemsize == 4 and out.is_floating_point(), "tri_edm: out must be float32 CUDA")
    _ok(lib().tri_edm(ctypes.byref(m), _strategy(strategy), _ptr(pts), pts.shape[1], pts.stride(0),
                      _cap(pts), _ptr(out), _nbytes(out),
                      _stream(stream)), "tri_edm")


def tri_edm_host(m: TriMap, strategy, h_pts, d_pts_ws, h_out, d_ws, band_cells=0):
    """Host-buffer EDM (synchronous): h_pts/h_out CPU tensors (pinned for overlap)."""
    _need(not h_pts.is_cuda and h_pts.dtype.itemsize == 4 and h_pts.is_floating_point() and h_pts.dim() == 2
          and h_pts.stride(1) == 1, "tri_edm_host: h_pts must be an (n, dim) float32 host tensor")
    _need(not h_out.is_cuda and h_out.dtype.itemsize == 4 and h_out.is_floating_point(),
          "tri_edm_host: h_out must be a float32 host tensor")
    _need(d_pts_ws.is_cuda and d_ws.is_cuda, "tri_edm_host: d_pts_ws and d_ws must be CUDA tensors")
    _ok(lib().tri_edm_host(ctypes.byref(m), _strategy(strategy), _ptr(h_pts), h_pts.shape[1], h_pts.stride(0),
                           _cap(h_pts), _ptr(d_pts_ws), _nbytes(d_pts_ws), _ptr(h_out), _nbytes(h_out),
                           _ptr(d_ws), _nbytes(d_ws), band_cells), "tri_edm_host")


def tri_collide_workspace_size(m: TriMap, strategy) -> int:
    return int(lib().tri_collide_workspace_size(ctypes.byref(m), _strategy(strategy)))


_collide_ws = {}


def collide_workspace(m: TriMap, strategy, device=None):
    """A cached device workspace of tri_collide_workspace_size bytes (None if 0): plain
    device memory the library reads and writes -- allocation is the caller's job."""
    nb = tri_collide_workspace_size(m, strategy)
    if nb == 0:
        return None
    import torch
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = (dev.index, nb)
    if key not in _collide_ws:
        _collide_ws.clear()
        _collide_ws[key] = torch.empty(nb, dtype=torch.uint8, device=dev)
    return _collide_ws[key]


def tri_tc_tf32_probe(x, y, d, stream=None):
    """Test hook: d (128 x 128 fp32) = x (128 x 8) @ y (128 x 8)^T on one tcgen05 tf32 MMA."""
    for t in (x, y, d):
        _need(t.is_cuda and t.dtype.itemsize == 4 and t.is_floating_point() and t.is_contiguous(),
              "tri_tc_tf32_probe: contiguous float32 CUDA tensors")
    _need(x.numel() == 1024 and y.numel() == 1024 and d.numel() == 16384, "tri_tc_tf32_probe: 128x8, 128x8, 128x128")
    _ok(lib().tri_tc_tf32_probe(_ptr(x), _ptr(y), _ptr(d), _stream(stream)), "tri_tc_tf32_probe")


def tri_tc_f16_probe(x, y, d, stream=None):
    """Test hook: d (128 x 128 fp16) = x (128 x 16 fp16) @ y (128 x 16 fp16)^T on one tcgen05
    kind::f16 MMA into an F16 accumulator."""
    for t in (x, y, d):
        _need(t.is_cuda and t.element_size() == 2 and t.is_contiguous(), "tri_tc_f16_probe: contiguous 16-bit CUDA")
    _need(x.numel() == 2048 and y.numel() == 2048 and d.numel() == 16384, "tri_tc_f16_probe: 128x16, 128x16, 128x128")
    _ok(lib().tri_tc_f16_probe(_ptr(x), _ptr(y), _ptr(d), _stream(stream)), "tri_tc_f16_probe")


def tri_collide(m: TriMap, strategy, spheres, count, stream=None, ws=None):
    """spheres: (n, 4) float32 CUDA tensor (x, y, z, r); count: 8-byte integer CUDA tensor (>= 1 elem).
    ws: the workspace of the tensor-core strategies (default: a cached one, collide_workspace)."""
    _need(spheres.is_cuda and spheres.dtype.itemsize == 4 and spheres.is_floating_point()
          and spheres.dim() == 2 and spheres.shape[1] == 4 and spheres.is_contiguous(),
          "tri_collide: spheres must be a contiguous (n, 4) float32 CUDA tensor")
    _need(count.is_cuda and count.element_size() == 8 and not count.is_floating_point(),
          "tri_collide: count must be an 8-byte integer CUDA tensor")
    if ws is None:
        ws = collide_workspace(m, strategy, spheres.device)
    _ok(lib().tri_collide(ctypes.byref(m), _strategy(strategy), _ptr(spheres), _nbytes(spheres), _ptr(count),
                          _nbytes(count), _ptr(ws), _nbytes(ws), _stream(stream)), "tri_collide")


def tri_ca_workspace_size(m: TriMap) -> int:
    return int(lib().tri_ca_workspace_size(ctypes.byref(m)))


def _u8(*ts):
    for t in ts:
        _need(t is None or (t.is_cuda and t.element_size() == 1), "CA buffers must be 1-byte CUDA tensors")


def tri_ca_step(m: TriMap, strategy, state_in, state_out, halo_above=None, halo_below=None, ws=None,
                stream=None):
    _u8(state_in, state_out, halo_above, halo_below)
    _ok(lib().tri_ca_step(ctypes.byref(m), _strategy(strategy), _ptr(state_in), _nbytes(state_in),
                          _ptr(state_out), _nbytes(state_out), _ptr(halo_above), _nbytes(halo_above),
                          _ptr(halo_below), _nbytes(halo_below), _ptr(ws), _stream(stream)), "tri_ca_step")


def tri_ca_steps(m: TriMap, strategy, k, state_in, state_out, halo_above=None, halo_below=None, ws=None,
                 stream=None):
    """k generations in one call; halos are the k packed rows on either side."""
    _u8(state_in, state_out, halo_above, halo_below)
    _ok(lib().tri_ca_steps(ctypes.byref(m), _strategy(strategy), int(k), _ptr(state_in), _nbytes(state_in),
                           _ptr(state_out), _nbytes(state_out), _ptr(halo_above), _nbytes(halo_above),
                           _ptr(halo_below), _nbytes(halo_below), _ptr(ws), _stream(stream)), "tri_ca_steps")


def _span(x):
    """Capacity of a halo given as a tensor; a raw address (peer / IPC memory) is sized by its owner."""
    if x is None:
        return 0
    return (1 << 62) if isinstance(x, int) else x.numel() * x.element_size()


def tri_ca_run_workspace_size(m: TriMap) -> int:
    return int(lib().tri_ca_run_workspace_size(ctypes.byref(m)))


def tri_ca_run(m: TriMap, strategy, steps, state_in, state_out, ws=None, stream=None):
    """`steps` generations on the bit-packed state (world 1, rho = 240); bytes in, bytes out.
    ws: tri_ca_run_workspace_size bytes of device memory (allocated here when None)."""
    _u8(state_in, state_out)
    if ws is None:
        import torch
        ws = torch.empty(tri_ca_run_workspace_size(m), dtype=torch.uint8, device=state_in.device)
    _ok(lib().tri_ca_run(ctypes.byref(m), _strategy(strategy), int(steps), _ptr(state_in), _nbytes(state_in),
                         _ptr(state_out), _nbytes(state_out), _ptr(ws), _nbytes(ws), _stream(stream)), "tri_ca_run")


def _addr(x):
    """A device address: a tensor's data pointer, a raw int (peer memory from tri_ipc_open), or None."""
    if x is None or isinstance(x, int):
        return x
    return x.data_ptr()


def tri_ca_steps_p2p(m: TriMap, strategy, k, state_in, state_out, halo_above=None, halo_below=None,
                     peer_above=None, peer_below=None, ws=None, stream=None):
    """tri_ca_steps that also stores its first / last k rows into the neighbours' halo
    buffers (peer_above / peer_below: addresses as include/tri.h defines them)."""
    _u8(state_in, state_out)
    _ok(lib().tri_ca_steps_p2p(ctypes.byref(m), _strategy(strategy), int(k), _ptr(state_in), _nbytes(state_in),
                               _ptr(state_out), _nbytes(state_out), _addr(halo_above), _span(halo_above),
                               _addr(halo_below), _span(halo_below), _addr(peer_above), _addr(peer_below),
                               _ptr(ws), _stream(stream)), "tri_ca_steps_p2p")


IPC_HANDLE_BYTES = 64


def tri_ipc_handle(t) -> tuple[bytes, int]:
    """(handle bytes, offset of t in its allocation) for another process's tri_ipc_open."""
    h = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    off = c_u64(0)
    _ok(lib().tri_ipc_handle(ctypes.c_void_p(_addr(t)), h, ctypes.byref(off)), "tri_ipc_handle")
    return h.raw, int(off.value)


def tri_ipc_open(handle: bytes, offset: int) -> tuple[int, int]:
    """Map another process's allocation: (address of the buffer, mapping base for tri_ipc_close)."""
    assert len(handle) == IPC_HANDLE_BYTES
    p, b = c_vp(), c_vp()
    _ok(lib().tri_ipc_open(handle, c_u64(offset), ctypes.byref(p), ctypes.byref(b)), "tri_ipc_open")
    return int(p.value), int(b.value)


def tri_ipc_close(base: int) -> None:
    _ok(lib().tri_ipc_close(ctypes.c_void_p(base)), "tri_ipc_close")


def tet_triplet(m: TetMap, strategy, pts4, energy, nu=1.0, stream=None):
    """pts4: contiguous (n, 4) float32 CUDA tensor; energy: float64 CUDA tensor of >= n elements."""
    _need(pts4.is_cuda and pts4.dtype.itemsize == 4 and pts4.is_floating_point() and pts4.dim() == 2
          and pts4.shape[1] == 4 and pts4.is_contiguous(), "tet_triplet: pts4 must be (n, 4) float32 CUDA")
    _need(energy.is_cuda and energy.element_size() == 8 and energy.is_floating_point(),
          "tet_triplet: energy must be a float64 CUDA tensor")
    _ok(lib().tet_triplet(ctypes.byref(m), _strategy(strategy), _ptr(pts4), _nbytes(pts4), float(nu),
                          _ptr(energy), _nbytes(energy), _stream(stream)), "tet_triplet")


def tri_last_launch_count() -> int:
    return int(lib().tri_last_launch_count())
