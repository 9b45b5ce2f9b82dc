"""GPU: the multi-rank fleet threshold (§8e) on one device.

The in-process communicator (enova_comm_create_local) runs `world` ranks as host
threads of this process, each with its own stream, through the SAME kernels and
collective sequence the NCCL path issues (3 histogram allreduces, an allgather
of tail counts, an allgather of fixed-size tail slots, the pack + fit launch).
The contract (include/enova.h, enova_fit_threshold): the result is bit-identical
on every rank and to the single-GPU fit of the rank-ordered concatenation.
The NCCL backend itself is covered at world size 1, inside a captured graph.
"""
import threading

import numpy as np
import pytest
import torch

from oracle import enova_oracle as O
from paper_2407_09486_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def E():
    from paper_2407_09486_b200 import build as B
    B.build()
    import paper_2407_09486_b200 as P
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return P


def run_ranks(world, fn):
    """fn(rank, stream) on `world` threads; returns the per-rank results (raises
    the first exception)."""
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                out[r] = fn(r, s)
            s.synchronize()
        except BaseException as e:   # noqa: BLE001 -- re-raised below
            err[r] = e

    import time
    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    deadline = time.monotonic() + 180
    for t in th:
        t.join(timeout=max(0.0, deadline - time.monotonic()))
        assert not t.is_alive(), "rank thread hung"
    for e in err:
        if e is not None:
            raise e
    return out


def shard(n, world, cuts):
    b = [0] + [int(c * n) for c in cuts] + [n]
    assert len(b) == world + 1
    return [(b[r], b[r + 1]) for r in range(world)]


@pytest.mark.parametrize("world,cuts", [(2, [0.5]), (3, [0.2, 0.9]), (4, [0.25, 0.25, 0.6])])
def test_local_comm_threshold_bit_identical(E, world, cuts):
    # uneven shards, one of them empty for world 4
    s = synth.score_mixture(400_000, seed=11 + world)
    sd = torch.from_numpy(s).cuda()
    single = E.fit_threshold(sd, 0.98, 1e-3)
    parts = shard(s.size, world, cuts)
    comms = E.Comm.create_local(world, 0)
    try:
        res = run_ranks(world, lambda r, st: E.fit_threshold(
            sd[parts[r][0]:parts[r][1]], 0.98, 1e-3, comm=comms[r], stream=st))
    finally:
        for c in comms:
            c.destroy()
    for r in range(world):
        assert res[r] == single, (r, res[r], single)
    o = O.pot_threshold(s, 0.98, 1e-3)
    assert single["t"] == o["t"] and single["n_peaks"] == o["n_peaks"]
    assert abs(single["z_q"] - o["z_q"]) <= 1e-9 * abs(o["z_q"])


def test_local_comm_all_peaks_on_one_rank(E):
    # every score above t lives on the last rank: its slot holds the whole tail
    s = np.sort(synth.score_mixture(300_000, seed=5))
    world = 3
    sd = torch.from_numpy(s).cuda()
    single = E.fit_threshold(sd, 0.98, 1e-3)
    parts = shard(s.size, world, [0.4, 0.8])
    comms = E.Comm.create_local(world, 0)
    n_global = s.size
    try:
        def rank(r, st):
            thr = E.fit_threshold_comm_async(sd[parts[r][0]:parts[r][1]], n_global, comms[r],
                                             0.98, 1e-3, stream=st)
            st.synchronize()
            return E.threshold_from_device(thr)
        res = run_ranks(world, rank)
    finally:
        for c in comms:
            c.destroy()
    for r in range(world):
        assert res[r] == single


def test_local_comm_too_few_exceedances_on_every_rank(E):
    s = np.zeros(20_000, np.float32)          # no score exceeds t
    sd = torch.from_numpy(s).cuda()
    comms = E.Comm.create_local(2, 0)
    try:
        def rank(r, st):
            try:
                E.fit_threshold(sd[r * 10_000:(r + 1) * 10_000], 0.98, 1e-3, comm=comms[r],
                                stream=st)
            except E.EnovaError as e:
                return e.name
            return "ok"
        res = run_ranks(2, rank)
    finally:
        for c in comms:
            c.destroy()
    assert res == ["ENOVA_ERR_TOO_FEW_EXCEEDANCES"] * 2


def _fleet(cfg_name="c1", n_inst=None, seed_off=3):
    cfg = synth.CONFIGS[cfg_name]
    W, M, H, Z = cfg["window"], cfg["n_metrics"], cfg["hidden"], cfg["latent"]
    N = n_inst or cfg["n_instances"]
    X = synth.metric_trace(N, cfg["n_steps"], M, seed=synth.DEFAULT_SEED + seed_off)
    wts = synth.detector_weights(W, M, H, Z, seed=synth.DEFAULT_SEED + seed_off)
    return X, wts


def test_local_comm_pipeline_matches_single_gpu(E):
    # the fleet's instances sharded over 3 ranks (uneven): every rank's flags /
    # scores / MD equal the single-GPU pipeline's rows, the threshold is identical
    X, wts = _fleet(n_inst=10)
    T = X.shape[1]
    tcal = T // 2
    det = E.PreparedDetector(wts)
    Xd = torch.from_numpy(X).cuda()
    ref = E.Pipeline(det, X.shape[0], T, tcal, overlap=False)   # the fit on the full grid,
    ref.enqueue(Xd)                                              # like the local ranks'
    r0 = ref.result()
    rows = [(0, 3), (3, 4), (4, 10)]
    comms = E.Comm.create_local(3, 0)
    try:
        def rank(r, st):
            a, b = rows[r]
            p = E.Pipeline(det, b - a, T, tcal, comm=comms[r])
            xs = Xd[a:b].contiguous()
            p.enqueue(xs, stream=st)
            st.synchronize()
            res = p.result()
            return (res.threshold, res.flags.cpu(), res.scores.cpu(), res.md.cpu())
        res = run_ranks(3, rank)
    finally:
        for c in comms:
            c.destroy()
    for r, (a, b) in enumerate(rows):
        thr, fl, sc, md = res[r]
        assert thr == r0.threshold
        assert torch.equal(fl, r0.flags[a:b].cpu())
        assert torch.equal(sc, r0.scores[a:b].cpu())
        assert torch.equal(md, r0.md[a:b].cpu())


def test_nccl_world1_pipeline_graph_matches_single_gpu(E):
    # the NCCL backend: the whole step, collectives included, captured in a graph
    X, wts = _fleet(n_inst=6, seed_off=4)
    T = X.shape[1]
    tcal = T // 2
    det = E.PreparedDetector(wts)
    Xd = torch.from_numpy(X).cuda()
    ref = E.Pipeline(det, X.shape[0], T, tcal)
    ref.enqueue(Xd)
    r0 = ref.result()
    comm = E.Comm.create(0, 1, torch.cuda.current_device())
    try:
        p = E.Pipeline(det, X.shape[0], T, tcal, comm=comm)
        p.capture(Xd)
        for _ in range(2):
            p.replay()
        res = p.result()
    finally:
        torch.cuda.synchronize()
        comm.destroy()
    assert res.threshold == r0.threshold
    assert torch.equal(res.flags, r0.flags)
    assert torch.equal(res.scores, r0.scores)


def test_local_comm_c2_scale_fleet_threshold(E):
    # the c2 calibration score vector (256 instances x 4937 windows, the bench's
    # threshold input size) sharded by instance over 4 ranks: bit-identical
    cfg = synth.CONFIGS["c2"]
    n_inst, per = cfg["n_instances"], cfg["n_steps"] // 2 - cfg["window"] + 1
    s = synth.score_mixture(n_inst * per, seed=21)
    sd = torch.from_numpy(s).cuda()
    single = E.fit_threshold(sd, 0.98, 1e-3)
    world = 4
    rows = [(r * n_inst // world) * per for r in range(world + 1)]
    comms = E.Comm.create_local(world, 0)
    try:
        res = run_ranks(world, lambda r, st: E.fit_threshold(
            sd[rows[r]:rows[r + 1]], 0.98, 1e-3, comm=comms[r], stream=st))
    finally:
        for c in comms:
            c.destroy()
    assert all(x == single for x in res)
    assert single["n"] == n_inst * per and single["n_peaks"] >= 10


def test_dead_peer_times_out_instead_of_hanging(E):
    """A rank that never reaches the collective (a dead peer): the waiting rank's
    fleet threshold returns ENOVA_ERR_NCCL once the communicator's timeout
    expires, the communicator is aborted, and every later call fails fast
    (include/enova.h failure handling; SURVEY §5 failure detection)."""
    import time
    comms = E.Comm.create_local(2)
    try:
        for c in comms:
            c.set_timeout(1.0)
        s = torch.from_numpy(synth.score_mixture(100_000, seed=5)).cuda()
        t0 = time.monotonic()
        with pytest.raises(E.EnovaError) as ei:
            E.fit_threshold(s, 0.98, 1e-3, comm=comms[0], n_global_max=200_000)   # rank 1 absent
        assert ei.value.name == "ENOVA_ERR_NCCL"
        assert time.monotonic() - t0 < 30
        with pytest.raises(E.EnovaError) as ei:
            comms[0].sum_i64(1)
        assert ei.value.name == "ENOVA_ERR_NCCL"
        with pytest.raises(E.EnovaError) as ei:
            comms[0].set_timeout(0.0)
        assert ei.value.name == "ENOVA_ERR_INVALID_ARGUMENT"
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()


def test_nccl_world1_wait_ok(E):
    comm = E.Comm.create(0, 1, torch.cuda.current_device())
    try:
        comm.set_timeout(30.0)
        x = torch.ones(1 << 20, device="cuda")
        (x * 2).sum()
        comm.wait()                     # bounded wait on the current stream: returns
        assert comm.sum_i64(7) == 7
    finally:
        comm.destroy()


def _dist_fit(E, sd, parts, world, n_global, q0=0.98, q=1e-3):
    comms = E.Comm.create_local(world, 0)
    try:
        def rank(r, st):
            thr = E.fit_threshold_dist_async(sd[parts[r][0]:parts[r][1]], n_global, comms[r],
                                             q0, q, stream=st)
            st.synchronize()
            return E.threshold_from_device(thr)
        return run_ranks(world, rank)
    finally:
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("world,cuts", [(1, []), (2, [0.5]), (3, [0.2, 0.9]),
                                        (4, [0.25, 0.25, 0.6])])
def test_distributed_fit_matches_oracle_and_ranks_agree(E, world, cuts):
    """The distributed-fit variant (enova_fit_threshold_dist_async):
    each rank fits on its own tail with the pass totals all-gathered -- every
    rank gets the same threshold (bit for bit), t / N_t exact, z_q within the
    1e-9 parity tolerance of the oracle and of the replicated fit."""
    s = synth.score_mixture(400_000, seed=31 + world)
    sd = torch.from_numpy(s).cuda()
    parts = shard(s.size, world, cuts)
    res = _dist_fit(E, sd, parts, world, s.size)
    for r in range(1, world):
        assert res[r] == res[0], (r, res[r], res[0])
    single = E.fit_threshold(sd, 0.98, 1e-3)
    o = O.pot_threshold(s, 0.98, 1e-3)
    d = res[0]
    assert d["t"] == o["t"] and d["n_peaks"] == o["n_peaks"] and d["n"] == s.size
    assert abs(d["z_q"] - o["z_q"]) <= 1e-9 * abs(o["z_q"]), (d, o)
    assert abs(d["z_q"] - single["z_q"]) <= 1e-9 * abs(single["z_q"])
    assert d["method"] == single["method"]


def test_distributed_fit_large_tail_and_edge_cases(E):
    """c5-like tail (2M-score mixture -> 40k peaks, the certified fp32 grid
    path) on 3 ranks with every peak on the last rank; too few exceedances on
    every rank -> the same error on every rank."""
    s = np.sort(synth.score_mixture(2_000_000, seed=77))
    sd = torch.from_numpy(s).cuda()
    parts = shard(s.size, 3, [0.3, 0.6])
    res = _dist_fit(E, sd, parts, 3, s.size)
    assert res[0] == res[1] == res[2]
    o = O.pot_threshold(s, 0.98, 1e-3)
    assert res[0]["n_peaks"] == o["n_peaks"] and res[0]["t"] == o["t"]
    assert abs(res[0]["z_q"] - o["z_q"]) <= 1e-9 * abs(o["z_q"])
    z = torch.zeros(20_000, dtype=torch.float32, device="cuda")
    comms = E.Comm.create_local(2, 0)
    try:
        def rank(r, st):
            thr = E.fit_threshold_dist_async(z[r * 10_000:(r + 1) * 10_000], 20_000, comms[r],
                                             0.98, 1e-3, stream=st)
            st.synchronize()
            try:
                E.threshold_from_device(thr)
            except E.EnovaError as e:
                return e.name
            return "ok"
        st = run_ranks(2, rank)
    finally:
        for c in comms:
            c.destroy()
    assert st == ["ENOVA_ERR_TOO_FEW_EXCEEDANCES"] * 2


def test_distributed_fit_pipeline(E):
    """Sharded Pipelines with fit_mode='distributed' (3 in-process ranks, uneven
    shards): the same threshold on every rank, within 1e-9 of the single-GPU
    pipeline's; flags / scores / MD rows equal the single-GPU pipeline's
    (identical z_q in practice; asserted outside the R-19 band)."""
    X, wts = _fleet(n_inst=10, seed_off=9)
    T = X.shape[1]
    tcal = T // 2
    det = E.PreparedDetector(wts)
    Xd = torch.from_numpy(X).cuda()
    ref = E.Pipeline(det, X.shape[0], T, tcal, overlap=False)
    ref.enqueue(Xd)
    r0 = ref.result()
    rows = [(0, 3), (3, 4), (4, 10)]
    comms = E.Comm.create_local(3, 0)
    try:
        def rank(r, st):
            a, b = rows[r]
            p = E.Pipeline(det, b - a, T, tcal, comm=comms[r], fit_mode="distributed")
            p.enqueue(Xd[a:b].contiguous(), stream=st)
            st.synchronize()
            res = p.result()
            return (res.threshold, res.flags.cpu(), res.scores.cpu())
        res = run_ranks(3, rank)
    finally:
        for c in comms:
            c.destroy()
    z0 = r0.threshold["z_q"]
    for r, (a, b) in enumerate(rows):
        thr, fl, sc = res[r]
        assert thr == res[0][0]
        assert abs(thr["z_q"] - z0) <= 1e-9 * abs(z0)
        assert torch.equal(sc, r0.scores[a:b].cpu())
        far = (sc.double() - z0).abs() > 1e-3 * abs(z0)
        assert torch.equal(fl[far], r0.flags[a:b].cpu()[far])


def test_distributed_fit_nccl_world1_graph(E):
    """The NCCL backend with the distributed fit: the whole step (17 fit-step
    launches and the all-gathers between them) captured in one CUDA graph;
    equal to the eager distributed step bit for bit."""
    X, wts = _fleet(n_inst=6, seed_off=4)
    T = X.shape[1]
    tcal = T // 2
    det = E.PreparedDetector(wts)
    Xd = torch.from_numpy(X).cuda()
    comm = E.Comm.create(0, 1, torch.cuda.current_device())
    try:
        p = E.Pipeline(det, X.shape[0], T, tcal, comm=comm, fit_mode="distributed")
        p.enqueue(Xd)
        eager = p.result()
        th_e, fl_e = dict(eager.threshold), eager.flags.clone()
        p.capture(Xd)
        p.replay()
        g = p.result()
    finally:
        comm.destroy()
    assert g.threshold == th_e
    assert torch.equal(g.flags, fl_e)
    o = O.detect_pipeline(X, wts, tcal)
    assert abs(th_e["z_q"] - o["threshold"]["z_q"]) <= 1e-6 * abs(o["threshold"]["z_q"])
