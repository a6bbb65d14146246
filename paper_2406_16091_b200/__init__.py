"""paper_2406_16091_b200 -- B200-native (sm_100a) cutoff pair interactions on a cell grid
(arXiv 2406.16091 hot path).  Thin Python layer over the C ABI of libpi.so (include/pi.h):
torch provides device memory and streams; binning, scan, scatter, interactions and the
position update run in the library's CUDA kernels.
"""
from __future__ import annotations

import ctypes

import torch

from . import _lib as L

__all__ = ["Context", "PiError", "ALGOS", "KERNELS", "lib", "slab_info", "nccl_unique_id"]

ALGOS = L.ALGOS
KERNELS = L.KERNELS


def lib():
    return L.load()


class PiError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        name = L.STATUS_NAMES[status] if 0 <= status < len(L.STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {msg}")


def _config(dims, cell_width, r_c=None, origin=(0.0, 0.0, 0.0), kernel="gaussian", sigma=0.0, capacity=0,
            rank=0, nranks=1, x_subcells=0, lj=(0.0, 0.0, 0.0)):
    cfg = L.pi_config()
    for a in range(3):
        cfg.origin[a] = float(origin[a])
        cfg.dims[a] = int(dims[a])
    cfg.cell_width = float(cell_width)
    cfg.r_c = float(cell_width if r_c is None else r_c)
    cfg.kernel = L.KERNELS[kernel] if isinstance(kernel, str) else int(kernel)
    if cfg.kernel in (L.KERNELS["lj"], L.KERNELS["highflop"]):  # Lennard-Jones r, eps, E0 (0 -> r_c, 0, 1)
        for k in range(3):
            cfg.kparam[k] = float(lj[k])
    else:
        cfg.kparam[0] = float(sigma)
    cfg.capacity = int(capacity)
    cfg.rank = int(rank)
    cfg.nranks = int(nranks)
    cfg.x_subcells = int(x_subcells)
    return cfg


SLAB_KEYS = ("Lx", "gx_lo", "gx_hi", "nx_local", "gx_off", "own_lo", "own_hi", "msg_cap")


def slab_info(dims, cell_width, rank, nranks, capacity=0, r_c=None, **kw):
    """pi_slab_info: the X-slab of `rank` (a8).  Host only."""
    cfg = _config(dims, cell_width, r_c=r_c, capacity=capacity, rank=rank, nranks=nranks, **kw)
    if nranks > 1:
        cfg.nccl_unique_id = ctypes.c_void_p(1)  # only checked for presence
    out = (ctypes.c_int64 * 8)()
    st = L.load().pi_slab_info(ctypes.byref(cfg), out)
    if st != L.PI_OK:
        raise PiError(st, "pi_slab_info: invalid configuration")
    return dict(zip(SLAB_KEYS, (int(v) for v in out)))


def nccl_unique_id() -> bytes:
    """pi_nccl_unique_id: 128 bytes to broadcast to every rank before creating contexts."""
    buf = ctypes.create_string_buffer(128)
    st = L.load().pi_nccl_unique_id(buf)
    if st != L.PI_OK:
        raise PiError(st, "pi_nccl_unique_id failed")
    return buf.raw


def _ptr(t):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


class Context:
    """One libpi context on one GPU (pi_create / pi_destroy).

    dims, cell_width, origin: the cell grid (cell_width >= r_c);
    kernel: 'gaussian' | 'indicator' | 'candidate' | 'lj'; sigma: Gaussian width (0 -> r_c/3);
    lj: Lennard-Jones (r, eps, E0) of Eq. (1) (0 -> r_c, 0, 1);
    capacity: max particles resident.
    """

    def __init__(self, dims, cell_width, r_c=None, origin=(0.0, 0.0, 0.0), kernel="gaussian", sigma=0.0,
                 capacity=0, device=None, stream=None, rank=0, nranks=1, nccl_unique_id=None, x_subcells=0,
                 lj=(0.0, 0.0, 0.0)):
        self._lib = L.load()
        self.device = torch.device(device if device is not None else "cuda")
        self.dims = tuple(int(d) for d in dims)
        self.cell_width = float(cell_width)
        self.r_c = float(cell_width if r_c is None else r_c)
        self.origin = tuple(float(o) for o in origin)
        cfg = _config(self.dims, self.cell_width, self.r_c, self.origin, kernel, sigma, capacity, rank, nranks,
                      x_subcells, lj)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        cfg.stream = ctypes.c_void_p(stream.cuda_stream)
        self.rank, self.nranks = int(rank), int(nranks)
        self._uid = None
        if nccl_unique_id is not None:
            self._uid = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
            cfg.nccl_unique_id = ctypes.cast(self._uid, ctypes.c_void_p)
        self.cfg = cfg
        nbytes = self._lib.pi_workspace_bytes(ctypes.byref(cfg))
        if nbytes == 0:
            raise PiError(L.PI_EINVAL, "invalid configuration (pi_workspace_bytes returned 0)")
        self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        h = ctypes.c_void_p()
        st = self._lib.pi_create(ctypes.byref(cfg), _ptr(self.workspace), nbytes, ctypes.byref(h))
        if st != L.PI_OK:
            raise PiError(st, "pi_create failed")
        self._h = h
        self.capacity = int(capacity)
        self.n = 0
        self.slab = slab_info(self.dims, self.cell_width, self.rank, self.nranks, capacity, self.r_c)
        # local grid (X-slab with ghost layers when nranks > 1)
        self.local_dims = (self.slab["nx_local"], self.dims[1], self.dims[2])

    # ------------------------------------------------------------------ helpers
    def _check(self, st):
        if st != L.PI_OK:
            raise PiError(st, self._lib.pi_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._lib.pi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_tuning(self, xpencil_len=0, xpencil_cap=0, fullload_box=(0, 0, 0), fullload_cap=0, threads=0,
                   xpencil_slots=0, xpencil_targets=0, exchange_full=0, xpencil_layout=0, exchange_overlap=0):
        t = L.pi_tuning()
        t.xpencil_len, t.xpencil_cap, t.fullload_cap, t.threads = xpencil_len, xpencil_cap, fullload_cap, threads
        t.xpencil_slots = xpencil_slots
        t.xpencil_targets = xpencil_targets
        t.exchange_full = exchange_full
        t.xpencil_layout = xpencil_layout
        t.exchange_overlap = exchange_overlap
        for a in range(3):
            t.fullload_box[a] = int(fullload_box[a])
        self._check(self._lib.pi_set_tuning(self._h, ctypes.byref(t)))

    def _f32(self, t):
        assert t.device.type == "cuda" and t.dtype == torch.float32 and t.is_contiguous()
        return t

    # ------------------------------------------------------------------ ABI calls
    def bin(self, x, y, z, q, id=None):
        n = int(x.numel())
        for t in (x, y, z, q):
            self._f32(t)
        self._check(self._lib.pi_bin(self._h, n, _ptr(x), _ptr(y), _ptr(z), _ptr(q), _ptr(id)))
        self.n = n

    def interact(self, algo="auto", out=True):
        a = L.ALGOS[algo] if isinstance(algo, str) else int(algo)
        if out:
            phi, fx, fy, fz = (torch.empty(self.n, dtype=torch.float32, device=self.device) for _ in range(4))
            self._check(self._lib.pi_interact(self._h, a, _ptr(phi), _ptr(fx), _ptr(fy), _ptr(fz)))
            return phi, fx, fy, fz
        self._check(self._lib.pi_interact(self._h, a, None, None, None, None))
        return None

    def interact_into(self, algo, phi, fx, fy, fz):
        a = L.ALGOS[algo] if isinstance(algo, str) else int(algo)
        self._check(self._lib.pi_interact(self._h, a, _ptr(phi), _ptr(fx), _ptr(fy), _ptr(fz)))

    def step(self, algo="auto", dt=0.0):
        a = L.ALGOS[algo] if isinstance(algo, str) else int(algo)
        self._check(self._lib.pi_step(self._h, a, ctypes.c_float(dt)))

    def run_host(self, algo, x, y, z, q, phi, fx, fy, fz):
        """End-to-end call on host (CPU, ideally pinned) float32 tensors."""
        a = L.ALGOS[algo] if isinstance(algo, str) else int(algo)
        n = int(x.numel())
        self._check(self._lib.pi_run_host(self._h, a, n, _ptr(x), _ptr(y), _ptr(z), _ptr(q), _ptr(phi), _ptr(fx),
                                          _ptr(fy), _ptr(fz)))
        self.n = n

    def run_host_submit(self, algo, x, y, z, q, phi, fx, fy, fz):
        """Pipelined end-to-end run on host (pinned) float32 tensors: enqueued, not synchronised; keep the
        tensors alive and unread until run_host_wait() (three runs in flight, pi.h)."""
        a = L.ALGOS[algo] if isinstance(algo, str) else int(algo)
        n = int(x.numel())
        self._check(self._lib.pi_run_host_submit(self._h, a, n, _ptr(x), _ptr(y), _ptr(z), _ptr(q), _ptr(phi),
                                                 _ptr(fx), _ptr(fy), _ptr(fz)))
        self.n = n

    def run_host_wait(self):
        """Blocks until every submitted run's outputs are in host memory."""
        self._check(self._lib.pi_run_host_wait(self._h))

    def _slots(self):
        """Sorted slots (owned + ghosts)."""
        if self.nranks == 1:
            return self.n
        s = self.stats(check=False)
        return s["n_owned"] + s["n_ghost"]

    def get_binning(self):
        """cell_of (caller order of the last bin), counts, offsets (local grid), perm (sorted slot -> caller
        index, -1 on ghost slots)."""
        nc = self.local_dims[0] * self.local_dims[1] * self.local_dims[2]
        dev = self.device
        cell_of = torch.empty(self.n, dtype=torch.int32, device=dev)
        counts = torch.empty(nc, dtype=torch.int32, device=dev)
        offsets = torch.empty(nc + 1, dtype=torch.int32, device=dev)
        perm = torch.empty(self._slots(), dtype=torch.int32, device=dev)
        self._check(self._lib.pi_get_binning(self._h, _ptr(cell_of), _ptr(counts), _ptr(offsets), _ptr(perm)))
        return cell_of, counts, offsets, perm

    def get_offsets(self):
        nc = self.local_dims[0] * self.local_dims[1] * self.local_dims[2]
        offsets = torch.empty(nc + 1, dtype=torch.int32, device=self.device)
        counts = torch.empty(nc, dtype=torch.int32, device=self.device)
        self._check(self._lib.pi_get_binning(self._h, None, _ptr(counts), _ptr(offsets), None))
        return counts, offsets

    def get_particles(self):
        """Owned particles (sorted order when nranks == 1, unspecified otherwise) with the last outputs."""
        dev = self.device
        n = self.n if self.nranks == 1 else self.stats(check=False)["n_owned"]
        f = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(8)]
        ids = torch.empty(n, dtype=torch.int32, device=dev)
        x, y, z, q, phi, fx, fy, fz = f
        self._check(self._lib.pi_get_particles(self._h, _ptr(x), _ptr(y), _ptr(z), _ptr(q), _ptr(ids), _ptr(phi),
                                               _ptr(fx), _ptr(fy), _ptr(fz)))
        return dict(x=x, y=y, z=z, q=q, id=ids, phi=phi, fx=fx, fy=fy, fz=fz)

    def count_pairs(self):
        """P: cutoff pairs of the owned targets in the current sorted state (pi_count_pairs)."""
        v = ctypes.c_int64(0)
        self._check(self._lib.pi_count_pairs(self._h, ctypes.byref(v)))
        return int(v.value)

    def stats(self, check=True):
        s = L.pi_stats()
        st = self._lib.pi_get_stats(self._h, ctypes.byref(s))
        if check:
            self._check(st)
        d = {k: getattr(s, k) for k, _ in L.pi_stats._fields_ if k not in ("reserved", "phase_ms")}
        d["bin_ms"], d["interact_ms"], d["exchange_ms"], d["host_copy_ms"] = (float(v) for v in s.phase_ms)
        return d
