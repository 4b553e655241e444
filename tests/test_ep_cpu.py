"""Expert-parallel dispatch/combine bookkeeping over gloo (world 2 and 3, CPU).

The exchange, the plan and the ordering are the product code; the expert math and
the router are the CPU oracle injected in place of the CUDA kernels (test only).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_02715_b200.expert_parallel import ExpertParallelMoE, build_plan, shard_bounds
from paper_2604_02715_b200.geometry import ModelSpec
from paper_2604_02715_b200.streamed import ForwardSpec

N, L, H, F, K = 2, 8, 32, 48, 3
T = 5  # tokens per rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_fns(bounds, rank, words):
    from oracle import xpg_oracle as O

    pool = O.WordPool(N, L, H, F, words)
    first, count = bounds[rank]

    def route_fn(seed, n, layer, num_experts, k):
        return torch.from_numpy(O.route(seed, n, layer, num_experts, k).astype(np.int64))

    def expert_fn(layer, rows, offsets):
        rows = rows.to(torch.float32).numpy()
        out = np.zeros_like(rows)
        off = offsets.numpy()
        for e in range(count):
            a, b = off[e], off[e + 1]
            if b > a:
                gu = pool.tensor_f32(layer, first + e + 1, 1)
                dn = pool.tensor_f32(layer, first + e + 1, 2)
                out[a:b] = O.expert_rows(gu, dn, rows[a:b])
        return torch.from_numpy(out)

    def combine_fn(rows, index, top_k):
        inv = np.float32(1.0 / top_k)
        r = rows.numpy()
        idx = index.numpy()
        y = np.zeros((idx.shape[0], r.shape[1]), dtype=np.float32)
        for s in range(idx.shape[1]):
            ok = idx[:, s] >= 0
            y[ok] += r[idx[ok, s]] * inv
        return torch.from_numpy(y)

    return route_fn, expert_fn, combine_fn


def _shared_fn(words_shared):
    from oracle import xpg_oracle as O

    sp = O.SharedPool(N, 1, H, F, words_shared)

    def shared_fn(layer, x, y):
        # the GPU path feeds the rows as their hi/lo bf16 planes: float32 x to ~2^-17
        y += torch.from_numpy(O.expert_rows(sp.tensor_f32(layer, 1, 1), sp.tensor_f32(layer, 1, 2), x.numpy()))

    return shared_fn, sp


def _worker(rank, world, port, seed, q, shared=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
      try:
        from oracle import xpg_oracle as O

        words = O.synth_payload(N, L, H, F, 4)
        spec = ModelSpec(N, L, H, F)
        fwd = ForwardSpec(T, K, seed)
        bounds = shard_bounds(L, world)
        route_fn, expert_fn, combine_fn = _oracle_fns(bounds, rank, words)
        shared_fn = _shared_fn(O.synth_payload(N, 1, H, F, 5))[0] if shared else None
        moe = ExpertParallelMoE(spec, fwd, rank, world, route_fn=route_fn, expert_fn=expert_fn,
                                combine_fn=combine_fn, shared_fn=shared_fn)
        x_all = np.random.default_rng(seed).standard_normal((world * T, H), dtype=np.float32)
        x = torch.from_numpy(x_all[rank * T:(rank + 1) * T].copy())
        for layer in (1, 2):
            x = moe.forward(layer, x)
        q.put((rank, x.numpy()))
      except Exception as exc:  # surface worker failures instead of a queue timeout
        import traceback

        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shared", [(2, False), (3, False), (2, True)])
def test_ep_matches_single_gpu_oracle(world, shared):
    from oracle import xpg_oracle as O

    seed = 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, q, shared)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for r, v in got.items():
        assert not isinstance(v, str), v
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y = np.concatenate([got[r] for r in range(world)])
    # single-device oracle on the concatenated batch (the dispatch moves float32 rows)
    words = O.synth_payload(N, L, H, F, 4)
    pool = O.WordPool(N, L, H, F, words)
    a = np.random.default_rng(seed).standard_normal((world * T, H), dtype=np.float32)
    sp = _shared_fn(O.synth_payload(N, 1, H, F, 5))[1] if shared else None
    for layer in (1, 2):
        a = O.layer_forward(pool, layer, a, K, seed, shared=sp)
    assert O.rel_l2(y, a) < 1e-5


def test_plan_bookkeeping_is_consistent():
    from oracle import xpg_oracle as O

    world, Tloc, Lx, k = 4, 7, 10, 3
    bounds = shard_bounds(Lx, world)
    assert [n for _, n in bounds] == [3, 3, 2, 2]
    routes = torch.from_numpy(O.route(5, world * Tloc, 1, Lx, k).astype(np.int64))
    plans = [build_plan(routes, r, world, Tloc, bounds) for r in range(world)]
    for r in range(world):
        for d in range(world):
            assert plans[r].send_counts[d] == plans[d].recv_counts[r]
        assert plans[r].offsets[-1].item() == sum(plans[r].recv_counts)
        assert sorted(plans[r].ret_index.reshape(-1).tolist()) == list(range(Tloc * k))
    # every pair is sent exactly once, to the owner of its expert
    total = sum(sum(p.send_counts) for p in plans)
    assert total == world * Tloc * k


@pytest.mark.parametrize("world,Tloc,Lx,k", [(2, 5, 8, 2), (3, 7, 10, 3), (8, 4, 256, 8), (4, 1, 6, 6)])
def test_peer_exchange_positions_match_the_collective(world, Tloc, Lx, k):
    """The peer-memory exchange's row positions (build_plan's p2p_* / c_* fields), replayed
    on host arrays, land every row exactly where the collective path puts it: dispatch rows
    at the owner's expert-major position, combine rows at the sender's return position."""
    from oracle import xpg_oracle as O

    bounds = shard_bounds(Lx, world)
    routes = torch.from_numpy(O.route(9, world * Tloc, 1, Lx, k).astype(np.int64))
    plans = [build_plan(routes, r, world, Tloc, bounds) for r in range(world)]
    H = 4
    xs = [torch.arange(Tloc * H, dtype=torch.float32).reshape(Tloc, H) + 1000 * r for r in range(world)]
    # collective path: send buffers, all-to-all by counts, expert-major permutation
    sends = [xs[r].index_select(0, plans[r].send_rows) for r in range(world)]
    recv = []
    for d in range(world):
        parts = []
        for r in range(world):
            off = sum(plans[r].send_counts[:d])
            parts.append(sends[r][off:off + plans[r].send_counts[d]])
        recv.append(torch.cat(parts).index_select(0, plans[d].to_expert))
    # peer path: every rank scatters straight into the owners' windows
    win = [torch.full((int(plans[d].c_rank.numel()), H), float("nan")) for d in range(world)]
    for r in range(world):
        p = plans[r]
        for i in range(p.p2p_src_rows.numel()):
            win[int(p.p2p_dst_rank[i])][int(p.p2p_dst_row[i])] = xs[r][int(p.p2p_src_rows[i])]
    for d in range(world):
        assert torch.equal(win[d], recv[d])
    # combine: owner rows back to the senders' return buffers
    outs = [recv[d] * 2 + 1 for d in range(world)]  # stand-in expert outputs, expert-major
    ret_coll = []
    for r in range(world):
        parts = []
        for d in range(world):
            back = outs[d].index_select(0, plans[d].from_expert)
            off = sum(plans[d].recv_counts[:r])
            parts.append(back[off:off + plans[d].recv_counts[r]])
        ret_coll.append(torch.cat(parts))
    ret = [torch.full((Tloc * min(k, Lx), H), float("nan")) for _ in range(world)]
    for d in range(world):
        p = plans[d]
        for i in range(p.c_rank.numel()):
            ret[int(p.c_rank[i])][int(p.c_row[i])] = outs[d][i]
    for r in range(world):
        assert torch.equal(ret[r], ret_coll[r])
