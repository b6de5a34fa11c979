"""Time-sharded extended-FD apply across ranks (one process per GPU), DESIGN.md §6.

Rank r owns the time slices T_r (a contiguous piece of the colexicographic vector, time slowest).
The spatial mode products are local.  The arrowhead solve couples only the time entries of one
spatial eigen-index (fdsolve.cpp:31-63), so the time direction runs on spatial slabs S_q after an
all-to-all transpose, and a second all-to-all brings the result back:

  x_r (N_s x |T_r|) --space fwd--> y_r --pack blocks y_r[S_q, :]--> all_to_all -->
  z_q (|S_q| x n_t, the blocks land contiguously in rank order) --time--> z'_q -->
  all_to_all (blocks z'_q[:, T_r] are already contiguous) --unpack--> y'_r --space bwd--> s_r

The exchange is a real data dependency of the path (not an artefact): NCCL over NVLink on the GPU
box, gloo in the CPU tests.  Compute is delegated to a backend:
  * `DeviceBackend` -- the C ABI stages (stiga_fd_apply_space / _time, stiga_copy_blocks);
  * tests supply a CPU backend built on the oracle (tests/test_distributed.py).
"""
import ctypes
from dataclasses import dataclass
from typing import List

import numpy as np

from ._lib import check, lib


def partition(n, parts):
    """Balanced contiguous partition of range(n): (offsets, sizes); the first n % parts get +1."""
    base, extra = divmod(n, parts)
    sizes = [base + (1 if i < extra else 0) for i in range(parts)]
    offsets = [sum(sizes[:i]) for i in range(parts)]
    return offsets, sizes


@dataclass
class ShardPlan:
    world: int
    rank: int
    n_s: int  # spatial DoFs N_s
    n_t: int
    t_off: List[int]
    t_len: List[int]
    s_off: List[int]
    s_len: List[int]

    @staticmethod
    def make(dims, world, rank):
        n_s = int(np.prod(dims[:-1]))
        n_t = int(dims[-1])
        if n_t < world or n_s < world:
            raise ValueError("ShardPlan: fewer time slices or spatial indices than ranks")
        t_off, t_len = partition(n_t, world)
        s_off, s_len = partition(n_s, world)
        return ShardPlan(world, rank, n_s, n_t, t_off, t_len, s_off, s_len)

    @property
    def local_size(self):
        return self.n_s * self.t_len[self.rank]

    def local_slice(self):
        """Range of the global colex vector owned by this rank."""
        a = self.n_s * self.t_off[self.rank]
        return a, a + self.local_size

    def send_splits_fwd(self):
        ntl = self.t_len[self.rank]
        return [self.s_len[q] * ntl for q in range(self.world)]

    def recv_splits_fwd(self):
        nsl = self.s_len[self.rank]
        return [nsl * self.t_len[r] for r in range(self.world)]


class DeviceBackend:
    """Stages on the device through the C ABI; tensors are torch CUDA float64."""

    def __init__(self, P, stream=None):
        self.P = P
        self.stream = stream

    def _st(self):
        import torch

        s = self.stream or torch.cuda.current_stream()
        return ctypes.c_void_p(s.cuda_stream)

    def space(self, x, out, backward, t0, ntl):
        check(lib().stiga_fd_apply_space(self.P.handle, int(backward), t0, ntl, ctypes.c_void_p(x.data_ptr()),
                                         ctypes.c_void_p(out.data_ptr()), self._st()), "fd_apply_space")

    def time(self, z, out, s0, nsl):
        check(lib().stiga_fd_apply_time(self.P.handle, s0, nsl, ctypes.c_void_p(z.data_ptr()),
                                        ctypes.c_void_p(out.data_ptr()), self._st()), "fd_apply_time")

    def copy_blocks(self, src, src_off, sld, dst, dst_off, dld, rows, cols):
        check(lib().stiga_copy_blocks(ctypes.c_void_p(src.data_ptr() + 8 * src_off), sld,
                                      ctypes.c_void_p(dst.data_ptr() + 8 * dst_off), dld, rows, cols, self._st()),
              "copy_blocks")


class ShardedExtendedFD:
    """Time-sharded ExtendedFDPreconditioner::apply (fdsolve.cpp:155-164) over a process group."""

    def __init__(self, backend, dims, group=None, world=None, rank=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.backend = backend
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.plan = ShardPlan.make(list(dims), world, rank)
        self._bufs = None

    def _buffers(self, like):
        import torch

        pl = self.plan
        n_loc = pl.local_size
        n_slab = pl.s_len[pl.rank] * pl.n_t
        if self._bufs is None or self._bufs[0].device != like.device:
            mk = lambda n: torch.empty(n, dtype=torch.float64, device=like.device)  # noqa: E731
            self._bufs = (mk(n_loc), mk(n_loc), mk(n_slab), mk(n_slab))
        return self._bufs

    def apply(self, x_local, out=None):
        """x_local: this rank's time slab (N_s x |T_r| colex).  Returns the slab of P^-1 x."""
        pl = self.plan
        y, send, z, z2 = self._buffers(x_local)
        self.stage_forward(x_local)
        self._all_to_all(z, send, pl.recv_splits_fwd(), pl.send_splits_fwd())
        self.stage_time()
        self._all_to_all(send, z2, pl.send_splits_fwd(), pl.recv_splits_fwd())
        return self.stage_backward(out if out is not None else x_local.new_empty(x_local.shape))

    # The three local stages (split out so a single-process test can drive several virtual ranks).
    def stage_forward(self, x_local):
        """Spatial forward products, then pack y[S_q, :] (row stride N_s) into contiguous blocks."""
        pl, b = self.plan, self.backend
        y, send, _, _ = self._buffers(x_local)
        ntl, t0 = pl.t_len[pl.rank], pl.t_off[pl.rank]
        b.space(x_local, y, False, t0, ntl)
        off = 0
        for q in range(pl.world):
            b.copy_blocks(y, pl.s_off[q], pl.n_s, send, off, pl.s_len[q], ntl, pl.s_len[q])
            off += pl.s_len[q] * ntl
        return send

    def stage_time(self):
        """Time direction on this rank's spatial slab z (the forward blocks landed in rank order)."""
        pl = self.plan
        _, _, z, z2 = self._bufs
        self.backend.time(z, z2, pl.s_off[pl.rank], pl.s_len[pl.rank])
        return z2

    def stage_backward(self, out):
        """Unpack the returned blocks into y[S_q, :] and apply the spatial backward products."""
        pl, b = self.plan, self.backend
        y, send, _, _ = self._bufs
        ntl, t0 = pl.t_len[pl.rank], pl.t_off[pl.rank]
        off = 0
        for q in range(pl.world):
            b.copy_blocks(send, off, pl.s_len[q], y, pl.s_off[q], pl.n_s, ntl, pl.s_len[q])
            off += pl.s_len[q] * ntl
        b.space(y, out, True, t0, ntl)
        return out

    def _all_to_all(self, out, inp, out_splits, in_splits):
        if self.plan.world == 1:
            out.copy_(inp)
            return
        self.dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                    group=self.group)
