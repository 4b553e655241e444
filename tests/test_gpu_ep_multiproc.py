"""Expert parallelism with two ranks on one B200: two processes, each an
ExpertParallelRunner on its own expert shard (own ring, own compressed host pool, budget
plan with sub-layer windows + device tier).  Rows move either through the collective
(gloo, host-staged here; NCCL across GPUs) or through peer memory (PeerExchange: CUDA IPC
windows, scatter kernels, epoch flags -- the same code path as across NVLink).  The
concatenated outputs must equal the single-device resident model on the concatenated
batch."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SPEC = (3, 8, 128, 256)
T, K, SEED = 12, 2, 9


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, budget, transport, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            import paper_2604_02715_b200 as X
            from paper_2604_02715_b200.budget import plan_residency
            from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

            spec = X.ModelSpec(*SPEC)
            fwd = X.ForwardSpec(T, K, SEED)
            container = X.generate_synthetic_model(spec, SEED)
            x_all = np.random.default_rng(SEED).standard_normal((world * T, spec.hidden_dim), dtype=np.float32)
            runner = ExpertParallelRunner(spec, container, fwd, rank, world, host_codec=True, transport=transport)
            assert runner.transport == transport, runner.transport_note
            count = runner.shard[1]
            if budget is not None:
                eb = spec.expert_bytes
                ceb = runner.device_tier_bytes(count) / (spec.num_layers * count) * 1.002
                plan = plan_residency(spec.num_layers, count, eb, ceb, budget * spec.num_layers * count * eb,
                                      min_window_bytes=1)
                runner.apply_plan(plan)
            rep = runner.run(2, x_all[rank * T:(rank + 1) * T].copy())
            rep2 = runner.run(1, x_all[rank * T:(rank + 1) * T].copy())  # epochs keep counting across runs
            torch.cuda.synchronize()
            runner.close()
            assert rep2.page_fault is None
            q.put((rank, (rep.final_activations.cpu().numpy(), rep.page_fault, rep.violations)))
        except Exception:
            import traceback

            q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("budget,transport", [(None, "nccl"), (0.4, "nccl"), (None, "p2p"), (0.4, "p2p")])
def test_two_ranks_on_one_gpu_match_resident(budget, transport):
    import torch.multiprocessing as mp

    import paper_2604_02715_b200 as X
    from oracle import xpg_oracle as O

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, budget, transport, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    for r, v in got.items():
        assert not isinstance(v, str), v
        assert v[1] is None and v[2] == [], (r, v[1], v[2])
    y = np.concatenate([got[r][0] for r in range(world)])
    spec = X.ModelSpec(*SPEC)
    container = X.generate_synthetic_model(spec, SEED)
    x_all = np.random.default_rng(SEED).standard_normal((world * T, spec.hidden_dim), dtype=np.float32)
    base = X.resident_baseline(2, spec, container, X.ForwardSpec(world * T, K, SEED), acts=x_all.copy())
    assert O.rel_l2(y, base) <= 1e-3


def test_peer_exchange_world1_matches_resident():
    """PeerExchange with one rank (the scatter writes into its own window)."""
    import paper_2604_02715_b200 as X
    from oracle import xpg_oracle as O
    from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

    spec = X.ModelSpec(*SPEC)
    fwd = X.ForwardSpec(T, K, SEED)
    container = X.generate_synthetic_model(spec, SEED, shared_experts=1)
    x = X.initial_activations(spec, fwd, SEED)
    runner = ExpertParallelRunner(spec, container, fwd, 0, 1, host_codec=True, transport="p2p")
    rep = runner.run(2, x.copy())
    runner.close()
    assert rep.page_fault is None and rep.violations == []
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert O.rel_l2(rep.final_activations.cpu().numpy(), base) <= 1e-3


def test_ep_decode_session_matches_run():
    """ExpertParallelRunner.open_session: one decode iteration per step on fresh activations,
    the same result as run(1) on each input (world 1, peer windows)."""
    import torch

    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

    spec = X.ModelSpec(*SPEC)
    fwd = X.ForwardSpec(T, K, SEED)
    container = X.generate_synthetic_model(spec, SEED)
    runner = ExpertParallelRunner(spec, container, fwd, 0, 1, host_codec=True, transport="p2p")
    xs = [np.random.default_rng(s).standard_normal((T, spec.hidden_dim), dtype=np.float32) for s in (1, 2, 3)]
    want = [runner.run(1, x.copy()).final_activations.cpu().numpy() for x in xs]
    out = torch.empty((T, spec.hidden_dim), dtype=torch.float32).pin_memory()
    with runner.open_session(max_iterations=4) as sess:
        for x, w in zip(xs, want):
            got = sess.step(torch.from_numpy(x).pin_memory(), out=out)
            assert got.numpy().tobytes() == w.tobytes()
    runner.close()


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_ep_empty_step(transport):
    """T = 0 under EP: the step still pages and exchanges (epochs published with no rows)
    and returns an empty batch."""
    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

    spec = X.ModelSpec(*SPEC)
    fwd = X.ForwardSpec(0, K, SEED)
    container = X.generate_synthetic_model(spec, SEED)
    runner = ExpertParallelRunner(spec, container, fwd, 0, 1, host_codec=True, transport=transport)
    rep = runner.run(2, np.zeros((0, spec.hidden_dim), np.float32))
    runner.close()
    assert tuple(rep.final_activations.shape) == (0, spec.hidden_dim)
    assert rep.page_fault is None and rep.violations == []


def _fault_worker(rank, world, port, mode, q):
    import time

    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            import paper_2604_02715_b200 as X
            from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

            spec = X.ModelSpec(*SPEC)
            fwd = X.ForwardSpec(T, K, SEED)
            container = X.generate_synthetic_model(spec, SEED)
            x = np.random.default_rng(rank).standard_normal((T, spec.hidden_dim), dtype=np.float32)
            runner = ExpertParallelRunner(spec, container, fwd, rank, world, host_codec=True, transport="p2p")
            if mode == "fault" or rank == 1:
                sess = runner.open_session(max_iterations=1)
                if mode == "fault" and rank == 0:
                    from paper_2604_02715_b200._lib import call

                    call("xpgb_fault_set", runner.ctx.handle, 1 | (1 << 8) | (1 << 32))  # as a page fault would
                t0 = time.time()
                sess.step(x)
                rep = sess.close()
                q.put((rank, (rep.page_fault, time.time() - t0)))
            else:  # "silent": rank 0 joins the session's epoch agreement, then never steps
                runner.peer.agree_epoch()
                time.sleep(30)
                q.put((rank, (None, 0.0)))
            torch.cuda.synchronize()
        except Exception:
            import traceback

            q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["fault", "silent"])
def test_peer_fault_and_timeout_reach_every_rank(mode):
    """A rank whose step faulted raises its peers' fault words with the epoch (its rows are
    garbage), so the peer reports a fault instead of combining stale rows; a peer that never
    publishes makes the wait give up after 20 s with a fault, not a trap."""
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fault_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        if p.is_alive():
            p.kill()
    for r, v in got.items():
        assert not isinstance(v, str), v
    fault1, secs1 = got[1]
    assert fault1 is not None and "peer rank 0" in fault1, fault1
    if mode == "fault":
        assert got[0][0] is not None
        assert "faulted" in fault1
    else:
        assert "no epoch" in fault1 and secs1 >= 19.0
