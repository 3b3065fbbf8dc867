"""Device plumbing: the per-(mesh, quadrature) library context and array conversion.

torch is used only for device memory and the current CUDA stream; all arithmetic
of the hot path runs in libb200hydro.so.  Public API functions accept numpy
arrays or CUDA torch tensors and return the kind they were given (numpy in ->
numpy out, like the reference; CUDA tensors stay resident).
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np
import torch

from . import _lib
from .tensor_basis import eval_basis, gauss_lobatto_nodes

DEVICE = "cuda"


def is_torch(a) -> bool:
    return isinstance(a, torch.Tensor)


_NP = {torch.float64: np.float64, torch.uint8: np.uint8, torch.int64: np.int64}


def to_dev(a, dtype=torch.float64) -> torch.Tensor:
    """Contiguous CUDA tensor copy/view of a numpy array or tensor."""
    if isinstance(a, torch.Tensor):
        return a.to(device=DEVICE, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a), dtype=_NP[dtype])).to(DEVICE)


def like(t: torch.Tensor, ref):
    """Return t as the same kind of array as ref (numpy or torch)."""
    if isinstance(ref, torch.Tensor):
        return t
    return t.cpu().numpy()


def empty(shape, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=DEVICE)


class LibError(RuntimeError):
    pass


class DeviceContext:
    """One hx_ctx: mesh connectivity, restriction maps and basis tables on the device."""

    def __init__(self, mesh, quad):
        self.lib = _lib.load()
        p = mesh.order
        if quad.n != p + 2:
            raise ValueError(f"the B200 kernels are built for Q1D = p+2 = {p + 2}, got {quad.n}")
        if not 1 <= p <= 4:
            raise ValueError(f"the B200 kernels support orders 1..4, got {p}")
        self.dim, self.order, self.q1d = mesh.dim, p, quad.n
        self.thermo_order = max(p - 1, 0)
        self.ne, self.nn = mesh.num_elements, mesh.num_nodes
        self.nl = (p + 1) ** self.dim
        self.nq = quad.n**self.dim
        self.nt = max(p, 1) ** self.dim
        kin = eval_basis(gauss_lobatto_nodes(p), quad)
        tnodes = np.zeros(1) if self.thermo_order == 0 else gauss_lobatto_nodes(self.thermo_order)
        th = eval_basis(tnodes, quad)
        self._keep = [np.ascontiguousarray(mesh.node_dofmap, dtype=np.int64),
                      np.ascontiguousarray(kin.B), np.ascontiguousarray(kin.G),
                      np.ascontiguousarray(th.B), np.ascontiguousarray(quad.weights, dtype=float)]
        dm, B, G, Bt, w = self._keep
        desc = _lib.MeshDesc(self.dim, p, quad.n, self.thermo_order, self.ne, self.nn,
                             _lib.as_i64_ptr(dm), _lib.as_f64_ptr(B), _lib.as_f64_ptr(G),
                             _lib.as_f64_ptr(Bt), _lib.as_f64_ptr(w), torch.cuda.current_device())
        h = C.c_void_p()
        rc = self.lib.hx_create(C.byref(desc), C.byref(h))
        if rc != _lib.HX_OK:
            raise ValueError(f"hx_create failed with code {rc} (dim={self.dim}, p={p}, NE={self.ne})")
        self.h = h
        self._fin = weakref.finalize(self, self.lib.hx_destroy, h)

    def sync_stream(self):
        self.lib.hx_set_stream(self.h, _lib.current_stream_ptr())

    def check(self, rc, what):
        if rc != _lib.HX_OK:
            msg = self.lib.hx_last_error(self.h).decode(errors="replace")
            if rc == _lib.HX_EINVAL:
                raise ValueError(f"{what}: {msg}")
            raise LibError(f"{what} failed (code {rc}): {msg}")

    def layout(self) -> str:
        """'brick' (structured index-free CG kernels) or 'csr' (generic transpose map)."""
        return "brick" if self.lib.hx_layout(self.h) == 1 else "csr"

    def launches(self) -> int:
        return int(self.lib.hx_kernel_launches(self.h))


def context_for(mesh, quad) -> DeviceContext:
    """Cached device context of a mesh for a quadrature rule (rebuilt if the
    connectivity array object changes)."""
    cache = mesh.__dict__.setdefault("_hx_ctx", {})
    key = (quad.n, quad.points.tobytes())
    ctx = cache.get(key)
    if ctx is None:
        ctx = DeviceContext(mesh, quad)
        cache[key] = ctx
    return ctx
