"""CPU, world_size 2 over gloo: the multi-view data-parallel driver (paper_2404_03202_b200/dp.py).

Each rank runs its share of the views through an oracle-backed ViewEngine (test infrastructure:
the FP64 restatement stands in for the device so the host logic runs without a GPU); the flat
gradient buffers are summed with torch.distributed.all_reduce over gloo. Checks: replicas are
bit-identical after every step, and equal a single-process run that trains all the views of each
batch itself (batch = sum of per-view backward() gradients, then one adam_step)."""
import os
import socket

import numpy as np
import pytest

from paper_2404_03202_b200 import dp, scenes

W, H, N_VIEWS, STEPS, BATCH = 64, 32, 4, 3, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class OracleViewEngine:
    """ViewEngine backed by the C restatement (FP64), flat gradient layout in a torch tensor."""

    def __init__(self):
        import torch

        import pyoracle
        self.pyoracle = pyoracle
        self.oracle = pyoracle.load("port")
        self.cloud = scenes.random_cloud(np.random.default_rng(5), count=40)
        self.poses = [scenes.random_pose(np.random.default_rng(100 + v)) for v in range(N_VIEWS)]
        target = scenes.random_cloud(np.random.default_rng(6), count=40)
        self.targets = [self.oracle.render(target, p, W, H).rgb for p in self.poses]
        n, bc = self.cloud.n, self.cloud.basis_count
        self.shapes = [("d_position", (n, 3)), ("d_sh", (n, bc, 3)), ("d_rotation", (n, 4)),
                       ("d_log_scale", (n, 3)), ("d_opacity_logit", (n,))]
        self.size = sum(int(np.prod(s)) for _, s in self.shapes)
        self.flat = torch.zeros(self.size, dtype=torch.float64)
        self.state = pyoracle.AdamState.zeros(n, bc)
        self.cfg = pyoracle.AdamConfig(iterations=100)
        self._reset_stats()

    def _reset_stats(self):
        """GradientBuffer screen stats + DensifyStats (resized, i.e. zeroed, by densify)."""
        import torch
        n = self.cloud.n
        self.norm_sum = torch.zeros(n, dtype=torch.float64)
        self.hits = torch.zeros(n, dtype=torch.int64)
        self.max_radius = torch.zeros(n, dtype=torch.float64)

    def stat_tensors(self):
        return [(self.norm_sum, "sum"), (self.hits, "sum"), (self.max_radius, "max")]

    def moment_tensors(self):
        import torch
        if getattr(self, "mflat", None) is None:
            st = self.state
            self.mflat = torch.from_numpy(np.concatenate([getattr(st, "m" + f).ravel() for f in
                                                          ("_position", "_sh", "_rotation", "_scale", "_opacity")]))
            self.vflat = torch.from_numpy(np.concatenate([getattr(st, "v" + f).ravel() for f in
                                                          ("_position", "_sh", "_rotation", "_scale", "_opacity")]))
        return self.mflat, self.vflat

    def _load_flat_moments(self):
        if getattr(self, "mflat", None) is None:
            return
        o = 0
        for f, (_, shape) in zip(("_position", "_sh", "_rotation", "_scale", "_opacity"), self.shapes):
            sz = int(np.prod(shape))
            setattr(self.state, "m" + f, self.mflat.numpy()[o:o + sz].reshape(shape).copy())
            setattr(self.state, "v" + f, self.vflat.numpy()[o:o + sz].reshape(shape).copy())
            o += sz
        self.mflat = self.vflat = None

    def densify_and_prune(self, config, extent, seed, radius_prune_active):
        import torch
        self._load_flat_params()
        self._load_flat_moments()
        cloud, state, summary = self.oracle.densify_and_prune(
            self.cloud, self.norm_sum.numpy(), self.hits.numpy(), self.max_radius.numpy(), self.state, config,
            extent, seed, radius_prune_active)
        self.cloud, self.state = cloud, state
        n, bc = cloud.n, cloud.basis_count
        self.shapes = [("d_position", (n, 3)), ("d_sh", (n, bc, 3)), ("d_rotation", (n, 4)),
                       ("d_log_scale", (n, 3)), ("d_opacity_logit", (n,))]
        self.size = sum(int(np.prod(s)) for _, s in self.shapes)
        self.flat = torch.zeros(self.size, dtype=torch.float64)
        self.pflat = None
        self._reset_stats()
        return summary

    def reset_opacity(self, ceiling):
        self._load_flat_params()
        self.oracle.reset_opacity(self.cloud, ceiling)
        self.pflat = None

    # --- flat parameters in the gradient layout (the sharded optimizer all-gathers them)
    def _fields(self):
        return [("positions", "d_position"), ("sh", "d_sh"), ("rotations", "d_rotation"),
                ("log_scales", "d_log_scale"), ("opacity_logits", "d_opacity_logit")]

    def param_tensor(self):
        import torch
        if getattr(self, "pflat", None) is None:
            self.pflat = torch.from_numpy(self.params().copy())
        return self.pflat

    def _load_flat_params(self):
        if getattr(self, "pflat", None) is None:
            return
        arr, o = self.pflat.numpy(), 0
        for (cf, _), (_, shape) in zip(self._fields(), self.shapes):
            sz = int(np.prod(shape))
            setattr(self.cloud, cf, arr[o:o + sz].reshape(shape).copy())
            o += sz

    def adam_step_shard(self, iteration, begin, count):
        """Adam on the flat element range only: the full elementwise step on copies, then the shard's
        parameters / moments written back (other elements belong to other ranks)."""
        import copy
        self._load_flat_params()
        self._load_flat_moments()
        old_cloud, old_state = self.cloud.copy(), copy.deepcopy(self.state)
        self.adam_step(iteration)
        new = self.params()
        flat = self.param_tensor().numpy()
        flat[begin:begin + count] = new[begin:begin + count]
        # moments: keep this rank's shard of the new state, the old values elsewhere
        offs = 0
        for f, (_, shape) in zip(["m_position", "m_sh", "m_rotation", "m_scale", "m_opacity"], self.shapes):
            sz = int(np.prod(shape))
            lo, hi = max(begin, offs), min(begin + count, offs + sz)
            for pre in ("m", "v"):
                name = pre + f[1:]
                a_new = getattr(self.state, name).ravel()
                a_old = getattr(old_state, name).ravel().copy()
                if lo < hi:
                    a_old[lo - offs:hi - offs] = a_new[lo - offs:hi - offs]
                setattr(self.state, name, a_old.reshape(getattr(old_state, name).shape))
            offs += sz
        self.cloud = old_cloud

    def accumulate_view(self, v):
        import torch
        self._load_flat_params()
        f = self.oracle.render(self.cloud, self.poses[v], W, H, keep_handle=True)
        loss, d = self.oracle.loss(f.rgb, self.targets[v], 0.0, 0.0)
        g = self.oracle.backward(f, d, self.cloud, self.poses[v])
        self.oracle.free(f)
        self.flat += torch.from_numpy(np.concatenate([getattr(g, k).ravel() for k, _ in self.shapes]))
        # GradientBuffer screen statistics (gradients.cpp:180-183) and DensifyStats::observe
        self.norm_sum += torch.from_numpy(g.screen_norm_sum)
        self.hits += torch.from_numpy(g.screen_hits)
        r = np.zeros(self.cloud.n)
        r[f.gaussian_id] = f.radius
        self.max_radius.copy_(torch.maximum(self.max_radius, torch.from_numpy(r)))
        return loss

    def grad_tensor(self):
        return self.flat

    def adam_step(self, iteration):
        self._load_flat_params()
        self._load_flat_moments()
        arr = self.flat.numpy()
        parts, o = {}, 0
        for k, s in self.shapes:
            sz = int(np.prod(s))
            parts[k] = arr[o:o + sz].reshape(s).copy()
            o += sz
        n = self.cloud.n
        g = self.pyoracle.Grads(parts["d_position"], parts["d_sh"], parts["d_rotation"], parts["d_log_scale"],
                                parts["d_opacity_logit"], np.zeros((n, 2)), np.zeros(n),
                                np.zeros(n, dtype=np.int64))
        self.oracle.adam_step(self.cloud, g, self.state, self.cfg, 1.0, iteration)
        self.flat.zero_()

    def params(self):
        c = self.cloud
        return np.concatenate([c.positions.ravel(), c.sh.ravel(), c.rotations.ravel(), c.log_scales.ravel(),
                               c.opacity_logits.ravel()])


def _worker(rank, world, port, out_dir, sharded=False):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = OracleViewEngine()
    if sharded:
        import torch

        def reduce_scatter(t, begin, count):  # gloo has no reduce_scatter: allreduce, keep the shard
            dist.all_reduce(t)

        def all_gather(t, begin, count):
            parts = [torch.empty(count, dtype=t.dtype) for _ in range(world)]
            dist.all_gather(parts, t[begin:begin + count].clone())
            t.copy_(torch.cat(parts))

        trainer = dp.DataParallelTrainer(eng, rank, world, reduce_scatter=reduce_scatter, all_gather=all_gather)
        assert trainer.sharded
    else:
        trainer = dp.DataParallelTrainer(eng, rank, world, allreduce=lambda t: dist.all_reduce(t))
    for step in range(STEPS):
        trainer.step(step + 1, dp.views_for_rank(step, BATCH, N_VIEWS, rank, world))
        if sharded:
            eng._load_flat_params()
        np.save(os.path.join(out_dir, f"rank{rank}_step{step}.npy"), eng.params())
    dist.barrier()
    dist.destroy_process_group()


def test_view_partition():
    assert dp.batch_views(0, 4, 16) == [0, 1, 2, 3]
    assert dp.batch_views(5, 4, 16) == [4, 5, 6, 7]
    assert dp.views_for_rank(1, 8, 16, 1, 4) == [9, 13]
    got = sorted(sum((dp.views_for_rank(3, 8, 16, r, 4) for r in range(4)), []))
    assert got == dp.batch_views(3, 8, 16) == sorted(dp.batch_views(3, 8, 16))
    with pytest.raises(ValueError):
        dp.DataParallelTrainer(object(), 0, 2, None)
    assert dp.shard_range(2360, 0, 2) == (0, 1180) and dp.shard_range(2360, 1, 2) == (1180, 1180)
    with pytest.raises(ValueError):
        dp.shard_range(2362, 0, 2)


@pytest.mark.parametrize("sharded", [False, True], ids=["replicated_adam", "sharded_adam"])
def test_two_rank_gloo_matches_single_process(tmp_path, oracle_port, sharded):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path), sharded), nprocs=2, join=True)
    single = OracleViewEngine()
    trainer = dp.DataParallelTrainer(single, 0, 1)
    for step in range(STEPS):
        trainer.step(step + 1, dp.batch_views(step, BATCH, N_VIEWS))
        r0 = np.load(tmp_path / f"rank0_step{step}.npy")
        r1 = np.load(tmp_path / f"rank1_step{step}.npy")
        assert np.array_equal(r0, r1), f"replicas diverged at step {step}"
        ref = single.params()
        # the allreduce sums the two ranks' partial sums: (g0 + g2) + (g1 + g3) vs ((g0 + g1) + g2) + g3
        assert np.allclose(r0, ref, rtol=1e-12, atol=1e-13), float(np.max(np.abs(r0 - ref)))


# ------------------------------------------------------------------ densification across ranks

DENSIFY_STEPS = 4
DENSIFY_AT = 2  # iteration (1-based) that densifies instead of stepping Adam (trainer.cpp:368-381)


def _densify_cfg():
    import pyoracle
    # thresholds low enough that the tiny scene clones, splits and prunes
    return pyoracle.DensifyConfig(densify_grad_threshold=1e-6, scale_split_threshold=0.3, prune_opacity=0.4)


def _densify_loop(trainer, eng, rank, world, out_dir=None):
    summaries = []
    for it in range(1, DENSIFY_STEPS + 1):
        views = dp.views_for_rank(it - 1, BATCH, N_VIEWS, rank, world)
        trainer.accumulate(views)
        if it == DENSIFY_AT:
            summaries.append(trainer.densify(_densify_cfg(), 1.0, 1234 + it, radius_prune_active=True))
        else:
            trainer.apply(it)
        eng._load_flat_params()
        eng._load_flat_moments()
        if out_dir:
            np.save(os.path.join(out_dir, f"d_rank{rank}_it{it}.npy"), eng.params())
            np.save(os.path.join(out_dir, f"d_rank{rank}_it{it}_m.npy"), eng.state.m_sh)
    return summaries


def _densify_worker(rank, world, port, out_dir, sharded):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "oracle"))
    import json

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    eng = OracleViewEngine()

    def reduce_stats(t, op):
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == "sum" else dist.ReduceOp.MAX)

    def all_gather(t, begin, count):
        parts = [torch.empty(count, dtype=t.dtype) for _ in range(world)]
        dist.all_gather(parts, t[begin:begin + count].clone())
        t.copy_(torch.cat(parts))

    if sharded:
        trainer = dp.DataParallelTrainer(eng, rank, world, reduce_scatter=lambda t, b, c: dist.all_reduce(t),
                                         all_gather=all_gather, reduce_stats=reduce_stats)
    else:
        trainer = dp.DataParallelTrainer(eng, rank, world, allreduce=lambda t: dist.all_reduce(t),
                                         reduce_stats=reduce_stats)
    summaries = _densify_loop(trainer, eng, rank, world, out_dir)
    with open(os.path.join(out_dir, f"d_rank{rank}_summary.json"), "w") as f:
        json.dump(summaries, f)
    dist.barrier()
    dist.destroy_process_group()


class _GroupedSingleProcess:
    """The 2-rank computation in one process: each 'rank' accumulates its own views' gradients and
    statistics from zero, and the partials are added (sum) / maxed exactly as the 2-rank collective
    does — so the replicas must equal it bit for bit."""

    def __init__(self, world):
        self.world = world
        self.eng = OracleViewEngine()

    def run(self):
        import torch
        eng, summaries = self.eng, []
        for it in range(1, DENSIFY_STEPS + 1):
            parts = []
            for r in range(self.world):
                eng.flat = torch.zeros(eng.size, dtype=torch.float64)
                eng._reset_stats()
                for v in dp.views_for_rank(it - 1, BATCH, N_VIEWS, r, self.world):
                    eng.accumulate_view(v)
                parts.append((eng.flat.clone(), eng.norm_sum.clone(), eng.hits.clone(), eng.max_radius.clone()))
            eng.flat = parts[0][0] + parts[1][0]
            eng.norm_sum, eng.hits = parts[0][1] + parts[1][1], parts[0][2] + parts[1][2]
            eng.max_radius = torch.maximum(parts[0][3], parts[1][3])
            if it == DENSIFY_AT:
                summaries.append(eng.densify_and_prune(_densify_cfg(), 1.0, 1234 + it, True))
            else:
                eng.adam_step(it)
            yield it, eng.params(), eng.state.m_sh, summaries


@pytest.mark.parametrize("sharded", [False, True], ids=["replicated_adam", "sharded_adam"])
def test_two_rank_densify_bit_equal_to_single_process(tmp_path, oracle_port, sharded):
    """A densify iteration across 2 gloo ranks: screen statistics summed, max radii maxed over
    ranks, (sharded) moments all-gathered, then densify_and_prune on every replica — replicas are
    bit-identical and equal the grouped single-process run bit for bit (parameters, moments, edit
    summary), and the edit really cloned / split / pruned."""
    import json

    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_densify_worker, args=(2, port, str(tmp_path), sharded), nprocs=2, join=True)
    for it, params, m_sh, summaries in _GroupedSingleProcess(2).run():
        r0 = np.load(tmp_path / f"d_rank0_it{it}.npy")
        r1 = np.load(tmp_path / f"d_rank1_it{it}.npy")
        assert np.array_equal(r0, r1), f"replicas diverged at iteration {it}"
        assert np.array_equal(r0, params), f"iteration {it} differs from the single process"
        if not sharded or it == DENSIFY_AT:  # sharded: moments outside a shard are stale until gathered
            assert np.array_equal(np.load(tmp_path / f"d_rank0_it{it}_m.npy"), m_sh), it
    s0 = json.load(open(tmp_path / "d_rank0_summary.json"))
    s1 = json.load(open(tmp_path / "d_rank1_summary.json"))
    assert s0 == s1 == summaries
    assert summaries[0]["cloned"] + summaries[0]["split"] > 0 and summaries[0]["pruned"] > 0, summaries
