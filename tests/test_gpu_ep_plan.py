"""The expert-parallel dispatch plan built on the GPU every step (DevicePlanner: the router
kernel + one plan CTA, xpgb_ep_plan) against the host restatement build_plan, and the EP
serving session routing afresh on every step.  Needs a B200."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,T,L,k", [(2, 5, 8, 2), (3, 7, 10, 3), (8, 4, 256, 8), (4, 1, 6, 6), (8, 256, 256, 8),
                                         (16, 3, 64, 4), (2, 0, 8, 2), (8, 64, 8, 2)])
def test_device_plan_equals_build_plan(world, T, L, k):
    import torch

    import paper_2604_02715_b200 as X
    from oracle import xpg_oracle as O
    from paper_2604_02715_b200.expert_parallel import DevicePlanner, build_plan, shard_bounds

    spec = X.ModelSpec(2, L, 64, 64)
    seed, layer = 13, 2
    fwd = X.ForwardSpec(T, k, seed)
    bounds = shard_bounds(L, world)
    routes = torch.from_numpy(O.route(seed, world * T, layer, L, k).astype(np.int64))
    kk = min(k, L)
    for rank in range(world):
        want = build_plan(routes, rank, world, T, bounds)
        got = DevicePlanner(spec, fwd, rank, world, T).plan(layer, T)
        torch.cuda.synchronize()
        n_own = int(want.c_rank.numel())
        assert int(got.counts[-1]) == n_own
        eq = lambda a, b: np.testing.assert_array_equal(np.asarray(a.cpu()).astype(np.int64), np.asarray(b).astype(np.int64))
        eq(got.p2p_src_rows, want.p2p_src_rows)
        eq(got.p2p_dst_rank, want.p2p_dst_rank)
        eq(got.p2p_dst_row, want.p2p_dst_row)
        eq(got.ret_index.reshape(-1), want.ret_index.reshape(-1))
        eq(got.offsets, want.offsets)
        eq(got.c_rank[:n_own], want.c_rank)
        eq(got.c_row[:n_own], want.c_row)
        got.resolve_counts()
        assert got.send_counts == want.send_counts and got.recv_counts == want.recv_counts
        eq(got.to_expert, want.to_expert)
        eq(got.from_expert, want.from_expert)
        assert T * kk == got.p2p_src_rows.numel()


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_session_routes_every_step(transport):
    """A serving session whose gate changes between steps (router_seed per step): every step
    equals the single-device resident stack routed with that step's seed, so nothing of an
    earlier step's routing is reused.  On the peer-memory transport a step also makes no
    synchronising torch call (torch sync debug mode "error")."""
    import torch

    import paper_2604_02715_b200 as X
    from oracle import xpg_oracle as O
    from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

    spec = X.ModelSpec(3, 8, 128, 256)
    T, K = 12, 2
    fwd = X.ForwardSpec(T, K, 5)
    container = X.generate_synthetic_model(spec, 5)
    runner = ExpertParallelRunner(spec, container, fwd, 0, 1, host_codec=True, transport=transport)
    seeds = [5, 77, 2**63 + 9, 5]
    xs = [np.random.default_rng(i).standard_normal((T, spec.hidden_dim), dtype=np.float32) for i in range(4)]
    outs = []
    with runner.open_session(max_iterations=len(seeds)) as sess:
        for x, s in zip(xs, seeds):
            xd = torch.from_numpy(x).cuda()
            torch.cuda.synchronize()
            if transport == "p2p":
                torch.cuda.set_sync_debug_mode("error")
            try:
                y = sess.step(xd, router_seed=s)
            finally:
                torch.cuda.set_sync_debug_mode("default")
            outs.append(y.cpu().numpy())
    runner.close()
    for x, s, y in zip(xs, seeds, outs):
        want = X.resident_baseline(1, spec, container, X.ForwardSpec(T, K, s), acts=x.copy())
        assert O.rel_l2(y, want) <= 1e-5, s
    assert O.rel_l2(outs[0], outs[1]) > 1e-2  # the gate really changed
