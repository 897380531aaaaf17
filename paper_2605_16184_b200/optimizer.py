# SPDX-License-Identifier: Apache-2.0
"""Torch-facing front end: one optimizer step over a list of fp32 CUDA
parameters, plus the owner-major parameter all-gather for block-sharded
multi-GPU runs.

PyTorch here is plumbing (device memory, streams, torch.distributed/NCCL);
every FLOP of the step runs in libasteria_b200.so.
"""
import ctypes as C

from . import abi
from .runtime import check, lib


# cudaStreamLegacy: the legacy default stream. torch reports its default stream
# as handle 0, which the C-ABI reads as "the blockset's own main stream" (a
# non-blocking stream that does not order with the legacy one), so handle 0 is
# passed as cudaStreamLegacy to keep torch's default-stream work ordered.
_CUDA_STREAM_LEGACY = 1


def stream_arg(stream):
    """C-ABI stream argument for a torch.cuda.Stream (or raw handle)."""
    sh = getattr(stream, "cuda_stream", stream)
    return C.c_void_p(sh if sh else _CUDA_STREAM_LEGACY)


class AsteriaOptimizer:
    """Shampoo / SOAP / KL-Shampoo step (harness.cpp:439-475 call order) over
    `params` with gradients `grads` (both lists of contiguous fp32 CUDA
    tensors of matching shapes; 1-D tensors are treated as 1 x n rows and get
    AdamW, harness.cpp:352)."""

    def __init__(self, params, grads, opt_cfg, sched_cfg=None, precision=abi.PREC_3XTF32,
                 rank=0, world=1, seed=1):
        import torch
        self.params, self.grads = list(params), list(grads)
        self.device = self.params[0].device
        for p, g in zip(self.params, self.grads):
            if p.dtype != torch.float32 or g.dtype != torch.float32 or not p.is_cuda or not g.is_cuda:
                raise abi.InvalidArgumentError("parameters and gradients must be fp32 CUDA tensors")
            if not p.is_contiguous() or not g.is_contiguous() or p.shape != g.shape:
                raise abi.ShapeMismatchError("parameters/gradients must be contiguous and shape-matched")
        self.opt = opt_cfg.copy()
        self.sched = (sched_cfg.copy() if sched_cfg is not None else abi.scheduler_defaults())
        self.sched.pf = self.opt.precondition_frequency
        self.rank, self.world = rank, world
        descs = (abi.ParamDesc * len(self.params))()
        for i, (p, g) in enumerate(zip(self.params, self.grads)):
            rows, cols = (p.shape[0], p.numel() // p.shape[0]) if p.dim() >= 2 else (1, p.numel())
            descs[i] = abi.ParamDesc(p.data_ptr(), g.data_ptr(), rows, cols, cols, cols)
        self._descs = descs
        h = C.c_void_p()
        check(lib.asg_blockset_create(self.device.index or 0, C.byref(self.opt), C.byref(self.sched), descs,
                                      len(self.params), precision, rank, world, seed, C.byref(h)))
        self._h = h
        s = C.c_void_p()
        check(lib.asg_blockset_stream(h, C.byref(s)))
        self.stream_handle = s.value
        self._gather_buf = None

    def __del__(self):
        if getattr(self, "_h", None):
            if getattr(self, "_nccl", None):
                lib.asg_set_allgather_comm(self._h, None, 1)
                lib.asg_nccl_comm_destroy(self._nccl)
                self._nccl = None
            lib.asg_blockset_destroy(self._h)
            self._h = None

    # ---- the step ----------------------------------------------------------
    def grad_sqnorm(self, stream=None):
        """Global squared gradient norm (read on `stream`, default torch's
        current stream, so gradient writes issued there are visible)."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        v, f = C.c_double(), C.c_int32()
        check(lib.asg_grad_sqnorm(self._h, stream_arg(stream), C.byref(v), C.byref(f)))
        if f.value:
            raise abi.NonFiniteError("non-finite gradient")
        return v.value

    @staticmethod
    def clip_scale_from_norm(norm, clip_norm=1.0):
        """clip_scale (harness.cpp:219-223)."""
        if norm <= clip_norm or norm == 0.0:
            return 1.0
        return clip_norm / norm

    def step(self, step, clip_scale=1.0, lr_scale=1.0, stream=None):
        """accumulate -> maybe_dispatch -> staleness_barrier -> precondition/apply
        -> StepEnd for every owned block. `stream` (a torch.cuda.Stream or raw
        handle; default: torch's current stream, like any torch op) is ordered
        before and after the step, so gradient writes issued on it before the
        call and parameter reads issued after it are race-free."""
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device)
        check(lib.asg_step(self._h, step, clip_scale, lr_scale, stream_arg(stream)))

    def synchronize(self):
        check(lib.asg_synchronize(self._h))

    def clock_advance(self, us):
        check(lib.asg_clock_advance(self._h, us))

    # ---- introspection -------------------------------------------------------
    @property
    def num_blocks(self):
        n = C.c_int64()
        check(lib.asg_blockset_num_blocks(self._h, C.byref(n)))
        return n.value

    def block_info(self, idx):
        i = abi.BlockInfo()
        check(lib.asg_blockset_block_info(self._h, idx, C.byref(i)))
        return i

    def read_block(self, idx, role):
        """One state tensor of owned block `idx` as fp64 host array (the
        per-block accessors of precond.hpp:63-75; parity checks)."""
        import numpy as np
        i = self.block_info(idx)
        m, n = i.spec.row_end - i.spec.row_begin, i.spec.col_end - i.spec.col_begin
        shape = {abi.FACTOR_L: (m, m), abi.FACTOR_R: (n, n), abi.INV_L: (m, m), abi.INV_R: (n, n),
                 abi.BASIS_L: (m, m), abi.BASIS_R: (n, n), abi.ROTATED_M: (m, n), abi.ROTATED_V: (m, n),
                 abi.KL_INV_L: (m, m), abi.KL_INV_R: (n, n), abi.EIGVALS_L: (m,), abi.EIGVALS_R: (n,)}[role]
        out = np.empty(shape)
        check(lib.asg_block_read(self._h, idx, role, out.ctypes.data_as(C.POINTER(C.c_double)), out.size))
        return out

    def stats(self):
        s = abi.PoolStats()
        check(lib.asg_get_stats(self._h, C.byref(s)))
        return s

    def freshness(self, idx):
        f = abi.Freshness()
        check(lib.asg_get_freshness(self._h, idx, C.byref(f)))
        return f

    def events(self):
        n = C.c_int64()
        check(lib.asg_get_events(self._h, None, 0, C.byref(n)))
        buf = (abi.Event * max(1, n.value))()
        check(lib.asg_get_events(self._h, buf, n.value, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def state_bytes(self):
        b = C.c_uint64()
        check(lib.asg_blockset_state_bytes(self._h, C.byref(b)))
        return b.value

    def attach_store(self, store):
        """F3: mirror every scheduler install's refreshed inverse state into a
        ``tierstore.TierStore`` (Host tier, prefetched toward Hot), as the
        reference's ShadowScheduler does with its store (asyncsched.cpp:164-184).
        The store must outlive the optimizer or be detached with ``None``."""
        self._store = store
        check(lib.asg_blockset_attach_store(self._h, store._h if store is not None else None))

    def on_hook(self, kind, step):
        """on_hook(ForwardPost / BackwardPre / StepEnd) asyncsched.cpp:223-286:
        ``abi.HOOK_FORWARD_POST`` drains staged transfers, ``abi.HOOK_BACKWARD_PRE``
        prefetches Cold inverse state to Host."""
        check(lib.asg_on_hook(self._h, kind, step))

    def synth_gradients(self, seed, step, stream=None):
        """Benchmark input: this rank's gradient slices <- N(0, 1/cols) from Philox keyed
        (seed, step, unit), one launch (asg_synth_gradients)."""
        check(lib.asg_synth_gradients(self._h, seed, step, stream_arg(stream)))

    def workspace_bytes(self):
        b = C.c_uint64()
        check(lib.asg_blockset_workspace_bytes(self._h, C.byref(b)))
        return b.value

    def profile(self, enable=True):
        check(lib.asg_profile_enable(self._h, 1 if enable else 0))

    def kernel_stats(self, reset=True):
        k = abi.KernelStats()
        check(lib.asg_get_kernel_stats(self._h, C.byref(k), 1 if reset else 0))
        return k

    def hbm_stats(self, reset=True):
        """HBM-bound kernels (prep, clip norm, AdamW) timed while profiling:
        {name: (launches, algorithmic bytes, ms)}."""
        h = abi.HbmStats()
        check(lib.asg_get_hbm_stats(self._h, C.byref(h), 1 if reset else 0))
        return {abi.HBM_NAMES[k]: (h.launches[k], h.bytes[k], h.ms[k]) for k in range(abi.HBM_KINDS)}

    # ---- multi-GPU ------------------------------------------------------------
    def shard_elems(self, rank):
        e = C.c_int64()
        check(lib.asg_shard_elems(self._h, rank, C.byref(e)))
        return e.value

    def gather_stride(self):
        e = C.c_int64()
        check(lib.asg_gather_stride(self._h, C.byref(e)))
        return e.value

    def reduce_scatter_grads(self, group=None):
        """Data-parallel gradients -> owners: every
        rank holds full local gradients; each rank receives the average over
        ranks of the blocks it owns (the reference's allreduce_avg,
        harness.cpp:425, restricted to what the owner needs) and writes it into
        its gradient tensors. One reduce-scatter of the owner-major buffer
        instead of an all-reduce of everything."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return
        stride = self.gather_stride()
        if getattr(self, "_rs_send", None) is None:
            self._rs_send = torch.zeros(stride * self.world, dtype=torch.float32, device=self.device)
            self._rs_recv = torch.zeros(stride, dtype=torch.float32, device=self.device)
        cur = torch.cuda.current_stream(self.device)
        check(lib.asg_pack_grads(self._h, C.c_void_p(self._rs_send.data_ptr()), stream_arg(cur)))
        if dist.get_backend(group) == "nccl":
            dist.reduce_scatter_tensor(self._rs_recv, self._rs_send, op=dist.ReduceOp.SUM, group=group)
        else:  # gloo (CPU test harness): stage through host memory
            send = self._rs_send.cpu()
            recv = torch.empty(stride, dtype=torch.float32)
            dist.reduce_scatter_tensor(recv, send, op=dist.ReduceOp.SUM, group=group)
            self._rs_recv.copy_(recv)
        check(lib.asg_unpack_reduced_grads(self._h, C.c_void_p(self._rs_recv.data_ptr()), 1.0 / self.world,
                                           stream_arg(cur)))

    def global_grad_sqnorm(self, group=None):
        """Global squared gradient norm after reduce_scatter_grads: the owned
        partial sums, all-reduced (the clip statistic, harness.cpp:219-223)."""
        import torch
        import torch.distributed as dist
        v, f = C.c_double(), C.c_int32()
        check(lib.asg_grad_sqnorm_owned(self._h, stream_arg(torch.cuda.current_stream(self.device)), C.byref(v),
                                        C.byref(f)))
        if f.value:
            raise abi.NonFiniteError("non-finite gradient")
        if self.world == 1:
            return v.value
        t = torch.tensor([v.value], dtype=torch.float64)
        if dist.get_backend(group) == "nccl":
            t = t.to(self.device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return float(t.item())

    def set_allgather_buckets(self, buckets_per_shape):
        """Bucketed all-gather layout (asg_set_allgather_buckets): allgather()
        then exchanges bucket by bucket."""
        check(lib.asg_set_allgather_buckets(self._h, buckets_per_shape))
        n = C.c_int64()
        check(lib.asg_bucket_count(self._h, C.byref(n)))
        self._buckets = []
        for b in range(n.value):
            st = C.c_int64()
            check(lib.asg_bucket_stride(self._h, b, C.byref(st)))
            self._buckets.append(st.value)

    def use_nccl(self, group=None, buckets_per_shape=4, fused=True):
        """This library's own NCCL communicator over the ranks (the 128-byte
        unique id is broadcast through torch.distributed when world > 1).
        fused: asg_step all-gathers bucket b while it updates bucket b+1
        (asg_set_allgather_comm); otherwise allgather() calls
        asg_allgather_params after the step."""
        import torch
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            check(lib.asg_nccl_unique_id(uid))
        if self.world > 1:
            import torch.distributed as dist
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.to(self.device)
            dist.broadcast(t, src=0, group=group)
            uid = (C.c_uint8 * 128)(*t.cpu().tolist())
        comm = C.c_void_p()
        check(lib.asg_nccl_comm_init(self.world, self.rank, uid, C.byref(comm)))
        self._nccl = comm
        self._nccl_fused = fused
        if fused:
            check(lib.asg_set_allgather_comm(self._h, comm, buckets_per_shape))
        else:
            self.set_allgather_buckets(buckets_per_shape)

    def close_nccl(self):
        if getattr(self, "_nccl", None):
            check(lib.asg_set_allgather_comm(self._h, None, 1))
            check(lib.asg_nccl_comm_destroy(self._nccl))
            self._nccl = None

    def allgather(self, group=None, stream=None):
        """All-gathers every rank's owned (updated) block slices of theta and
        scatters them back into the parameters. With use_nccl: the library's
        own NCCL collective (fused into the step, or asg_allgather_params
        here). Otherwise through torch.distributed: bucket by bucket after
        set_allgather_buckets, else one owner-major buffer; NCCL groups gather
        in HBM, gloo groups (CPU test harness) stage through host memory."""
        import torch
        import torch.distributed as dist
        if getattr(self, "_nccl", None):
            if not self._nccl_fused:
                check(lib.asg_allgather_params(self._h, self._nccl,
                                               stream_arg(stream or torch.cuda.current_stream(self.device))))
            return
        if self.world == 1:
            return
        if getattr(self, "_buckets", None):
            cur = torch.cuda.current_stream(self.device)
            cur.wait_stream(torch.cuda.ExternalStream(self.stream_handle))
            for b, stride in enumerate(self._buckets):
                send = torch.zeros(max(1, stride), dtype=torch.float32, device=self.device)
                check(lib.asg_bucket_pack(self._h, b, C.c_void_p(send.data_ptr()), stream_arg(cur)))
                if dist.get_backend(group) == "nccl":
                    recv = torch.empty(max(1, stride) * self.world, dtype=torch.float32, device=self.device)
                    dist.all_gather_into_tensor(recv, send, group=group)
                else:
                    r_cpu = torch.empty(max(1, stride) * self.world, dtype=torch.float32)
                    dist.all_gather_into_tensor(r_cpu, send.cpu(), group=group)
                    recv = r_cpu.to(self.device)
                if stride == 0:
                    continue
                check(lib.asg_bucket_unpack(self._h, b, C.c_void_p(recv.data_ptr()), stream_arg(cur)))
            return
        stride = self.gather_stride()
        if self._gather_buf is None:
            self._gather_send = torch.zeros(stride, dtype=torch.float32, device=self.device)
            self._gather_buf = torch.zeros(stride * self.world, dtype=torch.float32, device=self.device)
        # pack on the caller's stream once it has waited for the update: the
        # buffers' zero-fill (and any caller work) is ordered before the pack
        cur = torch.cuda.current_stream(self.device)
        cur.wait_stream(torch.cuda.ExternalStream(self.stream_handle))
        check(lib.asg_pack_owned(self._h, C.c_void_p(self._gather_send.data_ptr()), stream_arg(cur)))
        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(self._gather_buf, self._gather_send, group=group)
        else:
            send = self._gather_send.cpu()
            recv = torch.empty(stride * self.world, dtype=torch.float32)
            dist.all_gather_into_tensor(recv, send, group=group)
            self._gather_buf.copy_(recv)
        check(lib.asg_unpack_gathered(self._h, C.c_void_p(self._gather_buf.data_ptr()), stride,
                                      stream_arg(torch.cuda.current_stream(self.device))))
