"""The one-process-per-GPU path (RankSplitTrainer + NcclTransport), run as two
ranks sharing cuda:0 with the host-staged (gloo) collective: after several
split-parallel SGD steps both ranks hold identical parameters that match the
oracle's g=2 cooperative run (engine.py:95-647)."""

import os

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _setup():
    import paper_2303_13775_b200 as sg
    graph = sg.generate_powerlaw(8000, 80000, blocks=8, p_local=0.6, seed=2)
    pm = sg.range_partition(graph.num_vertices, 2)
    cache = sg.full_cache(pm)
    rng = np.random.default_rng(7)
    samples = [sg.sample_minibatch(graph, rng.choice(graph.num_vertices, 64, replace=False), [6, 4], rng)
               for _ in range(3)]
    return graph, pm, cache, samples


def _worker(rank, world, port, kind, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2303_13775_b200 as sg
        from paper_2303_13775_b200.engine import RankSplitTrainer
        torch.cuda.set_device(0)
        graph, pm, cache, samples = _setup()
        F, C = 12, 4
        feats_host = sg.synthetic_features(graph.num_vertices, F, seed=1)
        feats = sg.FeatureStore.from_host(feats_host, cache, devices=[rank])  # own shard only
        labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
        params = sg.init_params(kind, F, 8, C, 2, seed=3)
        tr = RankSplitTrainer(params, pm, cache, feats, labels, rank, world,
                              sg.NcclTransport(rank, world, stage_on_host=True))
        losses = []
        for s in samples:
            g = tr.step(s, 0.1)
            losses.append(float(g[tr.dp.n].item()))
        q.put((rank, losses, tr.dp.flat.cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["graphsage", "gat"])
def test_rank_local_path_two_processes(kind):
    from oracle.coop_oracle import CoopRun, reduce_and_sgd
    from oracle.model_oracle import glorot_params
    from oracle.split_oracle import split_sample
    import paper_2303_13775_b200 as sg
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 31000 + os.getpid() % 2000 + (7 if kind == "gat" else 0)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    import queue
    import time
    res, t0 = [], time.time()
    while len(res) < len(procs):
        try:
            res.append(q.get(timeout=5))
        except queue.Empty:
            dead = [p for p in procs if p.exitcode not in (None, 0)]
            assert not dead, f"a rank failed (exit codes {[p.exitcode for p in procs]})"
            assert time.time() - t0 < 300, "ranks timed out"
    res = sorted(res, key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
    (_, l0, p0), (_, l1, p1) = res
    assert np.array_equal(p0, p1)            # replicas identical after all-reduce + SGD
    assert l0 == l1
    graph, pm, cache, samples = _setup()
    F, C = 12, 4
    X = sg.synthetic_features(graph.num_vertices, F, seed=1).astype(np.float64)
    labels = sg.synthetic_labels(graph.num_vertices, C, seed=2)
    ref = glorot_params(kind, F, 8, C, 2, seed=3)
    for i, s in enumerate(samples):
        ws, wp = split_sample(s.layer_vertices, s.layer_edges, pm.assignment, 2, cache.cached)
        loss, grads = CoopRun(ref, ws, wp, X, labels).run()
        reduce_and_sgd(ref, grads, 0.1, len(s.targets))
        assert abs(l0[i] - loss) <= 1e-4 * abs(loss), (i, l0[i], loss)
    flat = np.concatenate([v.reshape(-1) for v in ref.values()])
    assert np.abs(p0 - flat).max() / np.abs(flat).max() < 1e-4
