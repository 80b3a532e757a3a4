"""Multi-view data parallelism for training.

One process per GPU. Every rank holds all N Gaussians, their gradients and Adam moments. A
training iteration over a batch of B views gives each rank its share of the views; each rank
accumulates the raw-parameter gradients of its views into its flat FP32 plane buffer (K4b adds,
never overwrites), the buffers are summed with ONE allreduce (NCCL over NVLink on the GPU box,
gloo in the CPU tests), and every rank applies the identical fused Adam step, so replicas stay
bit-identical.

Batch semantics (the reference trains one view per iteration, trainer.cpp:353-381): a batch of B
views = B reference backward() calls with their gradients summed, followed by one adam_step.

The single-view path has no exchange step and is never split across GPUs ("replicas only").
"""
from __future__ import annotations

from typing import Callable, Protocol, Sequence


def batch_views(step: int, views_per_step: int, n_views: int) -> list[int]:
    """The global batch of view ids for iteration `step` (0-based), cycling over the dataset."""
    return [(step * views_per_step + j) % n_views for j in range(views_per_step)]


def views_for_rank(step: int, views_per_step: int, n_views: int, rank: int, world: int) -> list[int]:
    """This rank's share of the batch: view j of the batch goes to rank j % world."""
    return batch_views(step, views_per_step, n_views)[rank::world]


class ViewEngine(Protocol):
    def accumulate_view(self, view_id: int) -> float | None: ...

    def grad_tensor(self): ...

    def adam_step(self, iteration: int) -> None: ...


def shard_range(size: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, begin + count) of a flat buffer of `size` elements owned by `rank` (equal shards,
    multiples of 4 elements so the fused Adam's float4 sweep stays aligned)."""
    if size % (4 * world):
        raise ValueError(f"flat size {size} is not a multiple of 4 x world ({world})")
    count = size // world
    return rank * count, count


class DataParallelTrainer:
    """Drives ViewEngine replicas: accumulate local views -> exchange -> Adam, plus the densify
    exchange of Trainer::run (trainer.cpp:353-381).

    Replicated optimizer (default): allreduce(sum) of the gradient buffer, then the identical fused
    Adam on every rank. Sharded optimizer (``reduce_scatter`` and ``all_gather`` given): each rank
    receives the summed gradients of its 1/world shard of the flat buffer, runs Adam on that shard
    only (engine.adam_step_shard) and the parameters are all-gathered — the same bytes on the wire
    as an allreduce, 1/world of the Adam traffic, and the same elementwise update (bit-identical to
    the replicated step for the same summed gradients). Moments outside a rank's shard are stale
    on that rank until :meth:`gather_optimizer_state` (done by :meth:`densify` before the edit).

    Densification (``reduce_stats(tensor, op)`` with op "sum" / "max"): the GradientBuffer screen
    statistics (gradients.cpp:180-183: sum of |dL/ds|, hit counts) and DensifyStats' max screen
    radius (trainer.cpp:180-186) are per-rank partials of the rank's views; they are summed / maxed
    over ranks, then every rank applies densify_and_prune with the same seed to identical inputs,
    so replicas stay bit-identical."""

    def __init__(self, engine: ViewEngine, rank: int, world: int, allreduce: Callable | None = None,
                 reduce_scatter: Callable | None = None, all_gather: Callable | None = None,
                 reduce_stats: Callable | None = None, force_shard: bool = False, native: bool = False):
        # native: the engine's context owns an NCCL communicator (Context.dp_init) and the library
        # issues every collective itself (osplat_gpu_dp_step; densify / save exchange inside)
        self.native = native
        if world > 1 and not native and allreduce is None and (reduce_scatter is None or all_gather is None):
            raise ValueError("world > 1 needs an allreduce or a reduce_scatter + all_gather pair")
        self.engine = engine
        self.rank = rank
        self.world = world
        self.allreduce = allreduce
        self.reduce_scatter = reduce_scatter
        self.all_gather = all_gather
        self.reduce_stats = reduce_stats
        # force_shard: take the sharded path even at world 1 (tests of the collective plumbing)
        self.sharded = (world > 1 or force_shard) and reduce_scatter is not None and all_gather is not None

    def accumulate(self, view_ids: Sequence[int]) -> float:
        """render -> loss -> backward (accumulate) of this rank's views (trainer.cpp:360-364)."""
        loss = 0.0
        for v in view_ids:
            out = self.engine.accumulate_view(v)
            if out is not None:
                loss += out
        return loss

    def apply(self, iteration: int) -> None:
        """Gradient exchange + Adam (trainer.cpp:381 for the batch's summed gradients)."""
        if self.native:
            self.engine.dp_step(iteration)
        elif self.sharded:
            grads = self.engine.grad_tensor()
            begin, count = shard_range(grads.numel(), self.rank, self.world)
            self.reduce_scatter(grads, begin, count)  # grads[begin:begin+count] <- sum over ranks
            self.engine.adam_step_shard(iteration, begin, count)
            self.all_gather(self.engine.param_tensor(), begin, count)  # every rank's shard -> all
        else:
            if self.world > 1:
                self.allreduce(self.engine.grad_tensor())
            self.engine.adam_step(iteration)

    def step(self, iteration: int, view_ids: Sequence[int]) -> float:
        loss = self.accumulate(view_ids)
        self.apply(iteration)
        return loss

    def gather_optimizer_state(self) -> None:
        """Sharded optimizer: all-gather the Adam moments so every rank holds all of them (before
        densify_and_prune, which carries moments per Gaussian, or a save of the sidecar)."""
        if not self.sharded or self.native:
            return
        for t in self.engine.moment_tensors():
            begin, count = shard_range(t.numel(), self.rank, self.world)
            self.all_gather(t, begin, count)

    def densify(self, config, extent: float, seed: int, radius_prune_active: bool) -> dict:
        """densify_and_prune (trainer.cpp:188-275) on every replica after the stats exchange; the
        caller skips this iteration's Adam step, as Trainer::run does (trainer.cpp:379-381)."""
        if self.world > 1 and not self.native:
            if self.reduce_stats is None:
                raise ValueError("densify at world > 1 needs reduce_stats")
            for t, op in self.engine.stat_tensors():
                self.reduce_stats(t, op)
        self.gather_optimizer_state()
        return self.engine.densify_and_prune(config, extent, seed, radius_prune_active)

    def reset_opacity(self, ceiling: float) -> None:
        self.engine.reset_opacity(ceiling)  # elementwise on identical replicas


class GpuViewEngine:
    """ViewEngine over a native.Context: render -> L1 loss -> backward(accumulate) per view on the
    device; the target images stay resident. Adam zeroes the gradients it consumes."""

    def __init__(self, ctx, poses, targets: dict, width: int, height: int, config, extent: float = 1.0,
                 mask_bottom_fraction: float = 0.0, lambda_ssim: float = 0.2, observe: bool = False):
        self.ctx = ctx
        self.poses = poses
        self.targets = targets  # view id -> device tensor (3*H*W float32, planar)
        self.W, self.H = width, height
        self.config = config
        self.extent = extent
        self.mask = mask_bottom_fraction
        self.lambda_ssim = lambda_ssim
        self.observe = observe  # DensifyStats::observe after every view (training with densification)
        self._wrap()

    def _wrap(self):
        """torch views (zero-copy) of the context's flat device buffers; re-taken after a
        densification edit (new planes, new stride)."""
        import torch
        v = self.ctx.view()
        flat = v.planes * v.stride
        dev = lambda ptr, n, ts="<f4": torch.as_tensor(_CudaArray(ptr, n, ts), device="cuda")
        self._grads, self._params = dev(v.grads, flat), dev(v.params, flat)
        self._m, self._v = dev(v.adam_m, flat), dev(v.adam_v, flat)
        self._stats = [(dev(v.screen_norm_sum, v.n, "<f8"), "sum"), (dev(v.screen_hits, v.n, "<i4"), "sum"),
                       (dev(v.max_radius_px, v.n), "max")]

    def accumulate_view(self, view_id: int):
        fr = self.ctx.render(self.poses[view_id], self.W, self.H)
        try:
            _, dimg = self.ctx.loss(fr, self.targets[view_id].data_ptr(), self.lambda_ssim, self.mask,
                                    want_value=False)
            self.ctx.backward_device(fr, dimg, accumulate=True)
            if self.observe:
                self.ctx.observe(fr)
        finally:
            fr.free()
        return None

    def grad_tensor(self):
        # the planes may be only *logically* zero (a consuming Adam step or zero_grad, and no view
        # of this rank accumulated since): osplat_gpu_view_buffers writes the zeros first, so a
        # rank without views contributes zeros to the collective, never last step's gradients
        self.ctx.view()
        return self._grads

    def adam_step(self, iteration: int):
        self.ctx.adam_step(self.config, self.extent, iteration, zero_grad=True)

    def dp_step(self, iteration: int):
        self.ctx.dp_step(self.config, self.extent, iteration)

    def adam_step_shard(self, iteration: int, begin: int, count: int):
        self.ctx.adam_step(self.config, self.extent, iteration, zero_grad=True, begin=begin, count=count)

    def param_tensor(self):
        return self._params

    def moment_tensors(self):
        return self._m, self._v

    def stat_tensors(self):
        """(tensor, reduction) of the per-Gaussian densification statistics: FP64 sum of |dL/ds|,
        int32 hit counts, FP32 max screen radius."""
        return self._stats

    def densify_and_prune(self, config, extent: float, seed: int, radius_prune_active: bool) -> dict:
        out = self.ctx.densify_and_prune(config, extent, seed, radius_prune_active)
        self._wrap()
        return out

    def reset_opacity(self, ceiling: float):
        self.ctx.reset_opacity(ceiling)


class _CudaArray:
    """__cuda_array_interface__ view of a device pointer (zero-copy torch interop)."""

    def __init__(self, ptr: int, n: int, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def nccl_stats_reduce(dist):
    """reduce_stats callable over torch.distributed: sum / max allreduce in place."""

    def reduce_stats(t, op):
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)

    return reduce_stats


def nccl_shard_collectives(dist):
    """reduce_scatter / all_gather callables over torch.distributed (NCCL on the GPU box), in place
    on the flat buffers: the rank's shard is a view of the full tensor."""

    def reduce_scatter(t, begin, count):
        dist.reduce_scatter_tensor(t[begin:begin + count], t)

    def all_gather(t, begin, count):
        dist.all_gather_into_tensor(t, t[begin:begin + count])

    return reduce_scatter, all_gather
