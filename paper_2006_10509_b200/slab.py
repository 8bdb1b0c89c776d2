"""Row-distributed Gerchberg-Saxton for one large plane (config C6).

One N x N run of ``run_gs`` (algorithms.py:147-202) split over G ranks (one
process per GPU, ``torch.distributed`` over NCCL; or G virtual ranks driven
from one process for tests). Rank r owns R = N/G lines of N points in the
"segmented row" layout of ``csrc/slab_kernels.cuh``: a torch tensor of shape
(G, R, R) whose block g is the chunk exchanged with rank g.

Per iteration (both GS passes are row passes, each followed by a corner turn):

    replay pass  (lines = original columns):  FFT -> error sums + amplitude projection -> IFFT
    turn         block transpose + all_to_all_single
    hologram pass (lines = original rows):    IFFT -> beam * x/|x| [-> snap] -> FFT
    turn

The start (random phase, row-major global draws) is a hologram pass; after the
loop one replay pass computes the final error and efficiency. Per-iteration
error sums stay on the device and are all-reduced once at the end (or every
iteration when ``progress``/``cancel`` hooks need live values). Each line is
transformed and projected with exactly the arithmetic of the single-GPU
generic passes, so index planes equal ``run_gs``'s; only the summation order
of the error sums differs.

torch provides the device buffers, the stream and the collectives (plumbing);
every pass and transpose is a kernel of ``libcghb200.so`` (``cgh_slab_*``).
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _native
from .algorithms import (
    BACKPROPAGATE,
    CANCELLED,
    COMPLETED,
    RANDOM_PHASE,
    RunReport,
    _check_inputs,
    _init_code,
    _mask_bytes,
)
from .errors import EmptyMaskError, NonFiniteError, UnsupportedShapeError, ZeroFieldError, ZeroTargetError
from .propagation import fill_propagation
from .runtime import current_device, runner_precision
from .slm import problem_for, states

SLAB_INIT, SLAB_HOLO, SLAB_GS, SLAB_FINAL, SLAB_INV, SLAB_FWD = 0, 1, 2, 3, 4, 6


def error_from_sums(sdd, srr, srd, denom, rescale):
    """Masked amplitude error from the four sums (passes.cuh error_from_sums,
    propagation.py:164-192)."""
    num = sdd
    if rescale and srr > 0.0:
        num = sdd - (srd * srd) / srr
    return num / denom


def local_inputs(cfg, target, illumination, world, rank, chunk_rows=1024):
    """This rank's share of the prepared inputs (host, fp64):

    * ``tgt``: R x N, ifftshifted |target| of columns [rR, (r+1)R), transposed,
      sign bit set outside the ifftshifted mask (propagation.py:164-192 on the
      uncentred replay plane);
    * ``beam``: R x N |illumination| of hologram rows [rR, (r+1)R) or None;
    * ``tcols``: R x N ifftshifted complex target columns (transposed), for
      the backpropagation start;
    * global statistics identical on every rank: count_in, denom = sum t^2
      over the mask, non-finite counts (accumulated over row chunks, so a
      16384^2 plane never needs a full-size temporary).

    ifftshift of an even-sized axis is a roll by -N/2, so shifted column v is
    original column (v + N/2) mod N and shifted row u is original row
    (u + N/2) mod N.
    """
    n = target.shape[0]
    rr = n // world
    r0 = rank * rr
    half = n // 2
    mask = np.asarray(cfg.metric.mask)
    if mask.shape != target.shape:
        _mask_bytes(cfg, target)   # raises DimensionMismatchError
    cols = (np.arange(r0, r0 + rr) + half) % n
    tcols = np.roll(target[:, cols], -half, axis=0)            # (N, R) = ifftshift(T)[:, r0:r0+R]
    mcols = np.roll(mask[:, cols] != 0, -half, axis=0)
    amp = np.abs(tcols)
    signed = np.where(mcols, amp, -amp)
    count_in, denom, nf_in, nf_all = 0, 0.0, 0, 0
    for a in range(0, n, chunk_rows):
        t = target[a:a + chunk_rows]
        m = mask[a:a + chunk_rows] != 0
        fin = np.isfinite(t)
        count_in += int(m.sum())
        denom += float(np.sum(np.abs(t[m]) ** 2))
        nf_in += int(np.count_nonzero(~fin & m))
        nf_all += int(np.count_nonzero(~fin))
    stats = {
        "count_in": count_in,
        "denom": denom,
        "nf_in": nf_in,
        "nf_all": nf_all,
        "nf_beam": 0 if illumination is None else int(np.count_nonzero(~np.isfinite(illumination))),
    }
    out = {
        "tgt": np.ascontiguousarray(signed.T, dtype=np.float64),
        "beam": None if illumination is None else np.ascontiguousarray(np.abs(illumination[r0:r0 + rr, :]), np.float64),
        "tcols": np.ascontiguousarray(tcols.T),
    }
    return out, stats


def to_segments(rows):
    """(R, N) row-major lines -> (G, R, R) segmented slab (numpy or torch)."""
    r, n = rows.shape
    g = n // r
    if isinstance(rows, np.ndarray):
        return rows.reshape(r, g, r).transpose(1, 0, 2)
    return rows.reshape(r, g, r).transpose(0, 1)


def from_segments(seg):
    """(G, R, R) segmented slab -> (R, N) row-major lines."""
    g, r, _ = seg.shape
    if isinstance(seg, np.ndarray):
        return seg.transpose(1, 0, 2).reshape(r, g * r)
    return seg.transpose(0, 1).reshape(r, g * r)


# ------------------------------------------------------------------ exchanges


def _fused_turn_targets(ranks_dst_ptrs, my_rank, block_bytes):
    """Destinations of this rank's G blocks for the fused corner turn: block g
    goes to rank g's receive buffer at chunk [my_rank]."""
    return [base + my_rank * block_bytes for base in ranks_dst_ptrs]


class LocalExchange:
    """G = 1: the corner turn is a plain transpose, no collective."""

    world = 1

    def alloc(self, ops, shape):
        return ops.empty(shape), ops.empty(shape)

    def turn(self, ranks, src, dst):
        r = ranks[0]
        s, d = getattr(r, src), getattr(r, dst)
        if hasattr(r.ops, "turn"):
            r.ops.turn(s, [d.data_ptr()])
        else:
            r.ops.transpose(s, d)

    def all_reduce(self, tensors):
        return tensors

    def gather(self, tensors):
        return tensors


class TorchExchange:
    """One rank of a torch.distributed group (NCCL on GPUs, gloo on CPU): the
    corner turn is block transposes into a send buffer + all_to_all_single."""

    needs_send_buffer = True

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def alloc(self, ops, shape):
        return ops.empty(shape), ops.empty(shape)

    def turn(self, ranks, src, dst):
        import torch

        (r,) = ranks
        r.ops.transpose(getattr(r, src), r.B)
        # complex slabs travel as (re, im) pairs: chunk g (R*R elements) -> rank g
        self.dist.all_to_all_single(torch.view_as_real(getattr(r, dst)), torch.view_as_real(r.B), group=self.group)

    def all_reduce(self, tensors):
        (t,) = tensors
        self.dist.all_reduce(t, group=self.group)
        return [t]

    def gather(self, tensors):
        import torch

        (t,) = tensors
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        return parts


class SymmetricExchange(TorchExchange):
    """One rank of a CUDA group with NVLink peer mappings (torch symmetric
    memory): the slab buffers live in one symmetric allocation, and the corner
    turn is ONE kernel per rank that transposes each block and stores it into
    the owning peer's buffer (cgh_slab_turn), followed by a device barrier.
    No NCCL on the data path."""

    needs_send_buffer = False

    def __init__(self, group=None):
        super().__init__(group)
        self.handle = None
        self.peer_base = None
        import torch.distributed._symmetric_memory as symm

        g = self.group if self.group is not None else self.dist.group.WORLD
        try:   # required before rendezvous on some torch versions, a no-op on others
            symm.enable_symm_mem_for_group(g.group_name)
        except Exception:  # noqa: BLE001
            pass

    def alloc(self, ops, shape):
        import torch.distributed._symmetric_memory as symm

        buf = symm.empty((2,) + tuple(shape), dtype=ops.cdtype, device=ops.device)
        group = self.group if self.group is not None else self.dist.group.WORLD
        self.handle = symm.rendezvous(buf, group)
        self.peer_base = list(self.handle.buffer_ptrs)
        self.half = buf[0].numel() * buf.element_size()      # byte offset of C inside the allocation
        self.block_bytes = buf[0, 0].numel() * buf.element_size()
        self.buf = buf
        return buf[0], buf[1]

    def turn(self, ranks, src, dst):
        (r,) = ranks
        off = 0 if dst == "A" else self.half
        r.ops.turn(getattr(r, src), _fused_turn_targets([b + off for b in self.peer_base], self.rank, self.block_bytes))
        self.handle.barrier(channel=0)


class _DevArray:
    """A raw device allocation seen by torch through __cuda_array_interface__
    (torch as a view, the library as the allocator: CUDA IPC handles must
    refer to allocation bases, which torch's caching allocator does not
    guarantee)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2, "strides": None}


class NcclExchange:
    """One rank of a distributed run whose data plane is the library's own
    (cgh_multi_*): the slab buffers are library allocations
    mapped into every peer with CUDA IPC, the corner turn is the fused
    peer-store kernel (cgh_slab_turn) followed by the device barrier on peer
    flags (cgh_multi_device_barrier), and the error sums / gathers are NCCL
    collectives of the library's communicator on the pass stream. torch.distributed
    only bootstraps: the broadcast of the NCCL id and the exchange of IPC
    handles (host objects)."""

    needs_send_buffer = False

    def __init__(self, group=None, device=None, stream=None):
        import torch
        import torch.distributed as dist

        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.lib = _native.library()
        if not self.lib.cgh_multi_available():
            raise RuntimeError("NCCL (libnccl.so.2) not available to the library")
        self.stream = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        idb = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _native.check(self.lib.cgh_multi_unique_id(idb))
        obj = [bytes(idb) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        idb = (ctypes.c_uint8 * 128).from_buffer_copy(obj[0])
        self.handle = ctypes.c_void_p()
        _native.check(self.lib.cgh_multi_create(self.device, self.world, self.rank, idb, ctypes.c_void_p(self.stream),
                                                ctypes.byref(self.handle)))
        self._allocs = []
        # barrier flags of every rank, mapped here
        flags = ctypes.c_void_p()
        _native.check(self.lib.cgh_multi_flags(self.handle, ctypes.byref(flags)))
        ptrs = self._exchange_ptr(flags.value)
        arr = (ctypes.c_void_p * self.world)(*[ctypes.c_void_p(p) for p in ptrs])
        _native.check(self.lib.cgh_multi_set_peer_flags(self.handle, arr))

    def _exchange_ptr(self, ptr):
        """Every rank's device pointer for `ptr`'s allocation, mapped into this
        process (own entry: `ptr` itself)."""
        h = (ctypes.c_uint8 * 64)()
        _native.check(self.lib.cgh_multi_ipc_handle(self.handle, ctypes.c_void_p(ptr), h))
        got = [None] * self.world
        self.dist.all_gather_object(got, bytes(h), group=self.group)
        out = []
        for g, hb in enumerate(got):
            if g == self.rank:
                out.append(ptr)
                continue
            p = ctypes.c_void_p()
            _native.check(self.lib.cgh_multi_ipc_open(self.handle, (ctypes.c_uint8 * 64).from_buffer_copy(hb),
                                                      ctypes.byref(p)))
            out.append(p.value)
        return out

    def alloc(self, ops, shape):
        import torch

        n = 1
        for d in shape:
            n *= int(d)
        esize = 16 if ops.cdtype == torch.complex128 else 8
        nbytes = 2 * n * esize
        ptr = ctypes.c_void_p()
        _native.check(self.lib.cgh_device_alloc(self.device, nbytes, ctypes.byref(ptr)))
        self._allocs.append(ptr.value)
        typestr = "<c16" if esize == 16 else "<c8"
        buf = torch.as_tensor(_DevArray(ptr.value, (2,) + tuple(shape), typestr), device=f"cuda:{self.device}")
        self.buf = buf
        self.half = n * esize                       # byte offset of C inside the allocation
        self.block_bytes = int(shape[1]) * int(shape[2]) * esize
        self.peer_base = self._exchange_ptr(ptr.value)
        return buf[0], buf[1]

    def turn(self, ranks, src, dst):
        (r,) = ranks
        off = 0 if dst == "A" else self.half
        r.ops.turn(getattr(r, src), _fused_turn_targets([b + off for b in self.peer_base], self.rank, self.block_bytes))
        _native.check(self.lib.cgh_multi_device_barrier(self.handle, ctypes.c_void_p(self.stream)))

    def all_reduce(self, tensors):
        (t,) = tensors
        _native.check(self.lib.cgh_multi_all_reduce_sum_f64(self.handle, ctypes.c_void_p(t.data_ptr()), t.numel(),
                                                             ctypes.c_void_p(self.stream)))
        return [t]

    def gather(self, tensors):
        import torch

        (t,) = tensors
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        _native.check(self.lib.cgh_multi_all_gather(self.handle, ctypes.c_void_p(t.data_ptr()),
                                                    ctypes.c_void_p(out.data_ptr()), t.numel() * t.element_size(),
                                                    ctypes.c_void_p(self.stream)))
        return list(out)

    def all_gather_into(self, out, t):
        """out (world, *t.shape) <- every rank's t (NCCL, pass stream)."""
        _native.check(self.lib.cgh_multi_all_gather(self.handle, ctypes.c_void_p(t.data_ptr()),
                                                    ctypes.c_void_p(out.data_ptr()), t.numel() * t.element_size(),
                                                    ctypes.c_void_p(self.stream)))

    def close(self):
        import torch

        if self.handle:
            torch.cuda.synchronize(self.device)
            self.lib.cgh_multi_destroy(self.handle)
            self.handle = ctypes.c_void_p()
        for p in self._allocs:
            self.lib.cgh_device_free(self.device, ctypes.c_void_p(p))
        self._allocs = []

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


class SimulatedExchange:
    """G virtual ranks in one process on one device (tests): phases run rank
    after rank and no kernel waits on another. With device ops the corner turn
    is the same fused kernel as SymmetricExchange, storing into the other
    virtual ranks' buffers (so its addressing is exercised here); otherwise
    transposes + block copies."""

    def __init__(self, world):
        self.world = world

    def alloc(self, ops, shape):
        return ops.empty(shape), ops.empty(shape)

    def turn(self, ranks, src, dst):
        if all(hasattr(r.ops, "turn") for r in ranks):
            bases = [getattr(r, dst).data_ptr() for r in ranks]
            for h, r in enumerate(ranks):
                s = getattr(r, src)
                r.ops.turn(s, _fused_turn_targets(bases, h, s[0].numel() * s.element_size()))
            return
        for r in ranks:
            r.ops.transpose(getattr(r, src), r.B)
        for h, r in enumerate(ranks):
            recv = getattr(r, dst)
            for g, q in enumerate(ranks):
                recv[g].copy_(q.B[h])

    def all_reduce(self, tensors):
        total = tensors[0].clone()
        for t in tensors[1:]:
            total += t
        return [total.clone() for _ in tensors]

    def gather(self, tensors):
        return list(tensors)


# ----------------------------------------------------------------- device ops


class NativeOps:
    """Slab passes and transposes through the C ABI (the product path)."""

    def __init__(self, cfg, n, world, rank, precision, device, stream):
        import torch

        self.torch = torch
        self.lib = _native.library()
        _native.require_device()
        self.pb, self._keep = problem_for(cfg.slm.scheme, n, n, precision, device)
        fill_propagation(self.pb, cfg.propagation)
        self.pb.rescale = 1 if cfg.metric.rescale else 0
        self.handle = ctypes.c_void_p()
        _native.check(self.lib.cgh_slab_create(ctypes.byref(self.pb), world, rank, ctypes.c_void_p(stream),
                                               ctypes.byref(self.handle)))
        self.device = torch.device("cuda", device)
        self.cdtype = torch.complex128 if precision == _native.FP64 else torch.complex64
        self.n_states = self.pb.n_states

    def close(self):
        if self.handle:
            self.lib.cgh_slab_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def empty(self, shape, kind="c"):
        t = self.torch
        dt = {"c": self.cdtype, "f64": t.float64, "idx": t.uint8 if self.n_states <= 256 else t.int32}[kind]
        return t.empty(shape, dtype=dt, device=self.device)

    def upload(self, arr, kind="c"):
        return self.torch.from_numpy(np.ascontiguousarray(arr)).to(self.device, self.cdtype if kind == "c" else None)

    def set_local(self, tgt, beam):
        _native.check(self.lib.cgh_slab_set_local(self.handle, _native.ptr(tgt), _native.ptr(beam)))

    def run(self, mode, data, gp=None, quantize=0, idx=None, sums=None):
        _native.check(self.lib.cgh_slab_pass(
            self.handle, mode, ctypes.c_void_p(data.data_ptr()), None if gp is None else ctypes.byref(gp),
            1 if quantize else 0, None if idx is None else ctypes.c_void_p(idx.data_ptr()),
            None if sums is None else ctypes.c_void_p(sums.data_ptr())))

    def transpose(self, src, dst):
        _native.check(self.lib.cgh_slab_transpose(self.handle, ctypes.c_void_p(src.data_ptr()),
                                                  ctypes.c_void_p(dst.data_ptr())))

    def turn(self, src, dst_ptrs):
        """Fused corner turn: transpose(src[g]) -> dst_ptrs[g] (device addresses)."""
        arr = (ctypes.c_void_p * len(dst_ptrs))(*[ctypes.c_void_p(int(p)) for p in dst_ptrs])
        _native.check(self.lib.cgh_slab_turn(self.handle, ctypes.c_void_p(src.data_ptr()), arr))

    def sync(self):
        self.torch.cuda.synchronize(self.device)


# ------------------------------------------------------------------ one rank


class SlabRank:
    """Buffers and passes of one rank: A (hologram slab), C (replay slab),
    B (send buffer, NCCL exchange only), the local index plane and the
    per-iteration sums."""

    def __init__(self, ops, world, n, iters, exch):
        self.ops = ops
        self.G, self.N, self.R = world, n, n // world
        shape = (world, self.R, self.R)
        self.A, self.C = exch.alloc(ops, shape)
        need_b = world > 1 and (getattr(exch, "needs_send_buffer", False) or not hasattr(ops, "turn"))
        self.B = ops.empty(shape) if need_b else None
        self.idx = ops.empty((self.R, n), "idx")
        self.sums = ops.empty((iters + 1, 4), "f64")
        self.sums.zero_()


def _turn(ranks, exch, src, dst):
    """Corner turn src -> dst on every rank (see the exchange classes)."""
    exch.turn(ranks, src, dst)


def _validate(stats, init_code, iters):
    # the single-GPU runner's order (runtime.cu gs_exec)
    if init_code == _native.INIT_BACKPROP and stats["nf_all"] > 0:
        raise NonFiniteError("target contains NaN or Inf")
    if stats["nf_beam"] > 0:
        raise NonFiniteError("illumination contains NaN or Inf")
    if stats["count_in"] == 0:
        raise EmptyMaskError("metric mask has no true pixels")
    if stats["denom"] == 0:
        raise ZeroTargetError("target is zero inside the mask")
    if stats["nf_in"] > 0 and iters > 0:
        raise NonFiniteError("target contains NaN or Inf inside the mask")


def drive(ranks, exch, cfg, local, gp, progress=None, cancel=None, stats=None):
    """Run the GS iterations over the given ranks (one real rank, or all the
    virtual ranks of a SimulatedExchange). Returns (sums (iters+1, 4) on the
    host after the all-reduce, iterations executed, cancelled flag)."""
    iters = max(0, int(cfg.iterations))
    qe = bool(cfg.quantize_each_iteration)
    init_code = _init_code(cfg.init_mode)

    def hologram_start(quantize):
        if init_code == _native.INIT_RANDOM:
            for r in ranks:
                r.ops.run(SLAB_INIT, r.A, gp, quantize, r.idx if quantize else None)
        else:   # backpropagate: ifftshift(T) -> inverse columns -> hologram pass
            for r, loc in zip(ranks, local):
                r.C.copy_(to_segments(r.ops.upload(loc["tcols"])))
                r.ops.run(SLAB_INV, r.C, gp)
            _turn(ranks, exch, "C", "A")
            for r in ranks:
                r.ops.run(SLAB_HOLO, r.A, gp, quantize, r.idx if quantize else None)
        _turn(ranks, exch, "A", "C")

    live = progress is not None or cancel is not None
    hologram_start(iters == 0)
    executed, stopped = 0, False
    for k in range(iters):
        if cancel is not None and _agree(exch, ranks, bool(cancel.is_set())):
            stopped = True
            break
        for r in ranks:
            r.ops.run(SLAB_GS, r.C, gp, sums=r.sums[k])
        if live and progress is not None:
            s = _reduced_row(exch, ranks, k)
            progress(k, error_from_sums(s[0], s[1], s[2], stats["denom"], cfg.metric.rescale))
        _turn(ranks, exch, "C", "A")
        last = k == iters - 1
        for r in ranks:
            r.ops.run(SLAB_HOLO, r.A, gp, qe or last, r.idx if last else None)
        _turn(ranks, exch, "A", "C")
        executed = k + 1
    if stopped:
        if executed == 0:
            hologram_start(True)
        else:   # A still holds the last hologram pass output (the turn only reads it)
            for r in ranks:
                r.ops.run(SLAB_HOLO, r.A, gp, True, r.idx)
            _turn(ranks, exch, "A", "C")
    for r in ranks:
        r.ops.run(SLAB_FINAL, r.C, gp, sums=r.sums[executed])
    totals = exch.all_reduce([r.sums for r in ranks])
    return totals[0].cpu().numpy(), executed, stopped


def _agree(exch, ranks, flag):
    """Cancel consensus: any rank's flag stops every rank."""
    if exch.world == 1 or isinstance(exch, SimulatedExchange):
        return flag
    import torch

    t = ranks[0].ops.empty((1,), "f64")
    t.fill_(1.0 if flag else 0.0)
    exch.all_reduce([t])
    return bool(t.item() > 0)


def _reduced_row(exch, ranks, k):
    rows = [r.sums[k].clone() for r in ranks]
    return exch.all_reduce(rows)[0].cpu().numpy()


class SlabSession:
    """Prepared distributed GS run: inputs partitioned and uploaded once, then
    ``run()`` repeatedly (benchmarks; the device work per run is the whole
    iteration loop). ``exchange``: None (G = 1), a ``TorchExchange`` (this
    process is one rank) or a ``SimulatedExchange`` (all ranks here)."""

    def __init__(self, cfg, target, illumination=None, *, exchange=None, precision=None, device=None,
                 ops_factory=None):
        target = np.asarray(target, dtype=np.complex128)
        _check_inputs(cfg, target, illumination)
        if cfg.init_mode not in (RANDOM_PHASE, BACKPROPAGATE):
            raise ValueError(f"unknown init_mode {cfg.init_mode!r}")
        self.init_code = _init_code(cfg.init_mode)
        h, w = target.shape
        if h != w:
            raise UnsupportedShapeError(f"slab runs need a square plane, got {target.shape}")
        self.cfg = cfg
        self.exch = exchange or LocalExchange()
        world = self.exch.world
        self.n = n = w
        self.iters = max(0, int(cfg.iterations))
        prec = runner_precision() if precision is None else precision
        dev = current_device() if device is None else device
        rank_ids = list(range(world)) if isinstance(self.exch, SimulatedExchange) else [getattr(self.exch, "rank", 0)]
        self.local, stats = [], None
        for rk in rank_ids:
            loc, stats = local_inputs(cfg, target, illumination, world, rk)
            self.local.append(loc)
        self.stats = stats
        _validate(stats, self.init_code, self.iters)
        if ops_factory is None:
            import torch

            stream = torch.cuda.current_stream(dev).cuda_stream

            def ops_factory(rk):
                return NativeOps(cfg, n, world, rk, prec, dev, stream)

        self.ranks = [SlabRank(ops_factory(rk), world, n, self.iters, self.exch) for rk in rank_ids]
        for r, loc in zip(self.ranks, self.local):
            r.ops.set_local(loc["tgt"], loc["beam"])

    def run(self, seed=None, progress=None, cancel=None):
        """One generation; returns (sums (iters+1, 4), executed, cancelled)."""
        cfg = self.cfg
        gp = _native.GsParams(self.iters, float(cfg.feedback_gain), 1 if cfg.quantize_each_iteration else 0,
                              self.init_code,
                              _native.Pcg64State.from_bitgen(np.random.PCG64(cfg.seed if seed is None else seed)))
        return drive(self.ranks, self.exch, cfg, self.local, gp, progress, cancel, self.stats)

    def errors(self, sums, executed):
        denom, rescale = self.stats["denom"], bool(self.cfg.metric.rescale)
        return [error_from_sums(s[0], s[1], s[2], denom, rescale) for s in sums[: executed + 1]]

    def indices(self, gather=True):
        if gather:
            parts = self.exch.gather([r.idx for r in self.ranks])
            return np.concatenate([p.cpu().numpy() for p in parts], axis=0)
        return np.concatenate([r.idx.cpu().numpy() for r in self.ranks], axis=0)

    def close(self):
        for r in self.ranks:
            close = getattr(r.ops, "close", None)
            if close:
                close()


def run_gs_slab(cfg, target, illumination=None, progress=None, cancel=None, *, exchange=None, gather=True,
                precision=None, device=None, ops_factory=None):
    """``run_gs`` over a row-slab decomposition (drop-in signature plus the
    distribution keywords). Returns (hologram, RunReport): the full complex128
    hologram when ``gather`` (every rank), else this rank's rows (R x N)."""
    start = time.perf_counter()
    sess = SlabSession(cfg, target, illumination, exchange=exchange, precision=precision, device=device,
                       ops_factory=ops_factory)
    try:
        sums, executed, stopped = sess.run(progress=progress, cancel=cancel)
        errs = sess.errors(sums, executed)
        s_fin = sums[executed]
        if s_fin[3] == 0.0:
            raise ZeroFieldError("replay field is zero")
        eff = s_fin[1] / s_fin[3]
        if progress is not None:
            progress(executed, errs[executed])
        idx = sess.indices(gather)
    finally:
        sess.close()
    holo = _native.expand_states(idx, states(cfg.slm.scheme))
    return holo, RunReport(
        error_trace=[(k, float(e)) for k, e in enumerate(errs)],
        final_error=float(errs[executed]),
        efficiency=float(eff),
        iterations_executed=int(executed),
        runtime_ms=(time.perf_counter() - start) * 1e3,
        seed_used=cfg.seed,
        termination=CANCELLED if stopped else COMPLETED,
    )
