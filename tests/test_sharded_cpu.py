"""Row-sharded solver host logic on CPU (gloo world_size 2; thread-emulated world 3).

``sharded_loop`` (paper_2201_12324_b200/sharded.py) is the multi-GPU loop of
SURVEY.md §8e.  Here it drives a float64 numpy *test double* of the device
engine (the CudaShardEngine contract: f half-step on the local rows, the
shard's column log2-partial, the rank-order combine, the fused check) through
real ``torch.distributed`` gloo collectives.  The sharded result must equal
the unsharded CPU oracle (oracle/, the reference restatement): same f (all
shards), g, iteration count, check trace and converged flag.
"""

import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2201_12324_b200.errors import DivergedError
from paper_2201_12324_b200.geometry import EpsilonSchedule
from paper_2201_12324_b200.sharded import ThreadComm, TorchComm, shard_rows, sharded_loop

LN2 = np.log(2.0)


class NumpyShardEngine:
    """float64 test double of CudaShardEngine (values in the kernel's log2 convention)."""

    def __init__(self, x_local, y, a_local, b):
        # explicit cost block: like the kernels, the double never validates its inputs
        self.C = oracle.PointCloudOracle(np.asarray(x_local, float), np.asarray(y, float)).cost_matrix()
        self.a = np.asarray(a_local, float)
        self.b = np.asarray(b, float)
        with np.errstate(divide="ignore"):
            self.la, self.lb = np.log(self.a), np.log(self.b)
        self.n, self.m = len(self.a), len(self.b)
        self.f = [np.zeros(self.n), np.zeros(self.n)]
        self.g = np.zeros(self.m)
        self.bias_f, self.bias_eps = None, None   # the potential the next cols half-step reads
        self.first_bad = 2 ** 31 - 1
        self.device = "cpu"

    @staticmethod
    def _bad(v):
        return bool(np.isnan(v).any() or np.any(v == np.inf))

    def set_g(self, g_init, kappa):
        self.g = np.zeros(self.m) if g_init is None else np.asarray(g_init, float).copy()
        if self._bad(self.g):
            self.first_bad = min(self.first_bad, 1)

    def rows(self, kappa, eps, kappa_next, which, step):
        with np.errstate(all="ignore"):
            lse = eps * oracle.logsumexp((self.g[None, :] - self.C) / eps, axis=1)
            self.f[which] = eps * self.la - lse
        self.bias_f, self.bias_eps = self.f[which], eps
        if self._bad(self.f[which]):
            self.first_bad = min(self.first_bad, step)

    def cols_partial(self, kappa):
        eps = self.bias_eps
        with np.errstate(all="ignore"):
            lse = oracle.logsumexp((self.bias_f[:, None] - self.C) / eps, axis=0)
        return torch.from_numpy(lse / LN2)

    def cols_finalize(self, lall, eps, kappa_next, step):
        L = lall.numpy()
        with np.errstate(all="ignore"):
            self.g = eps * self.lb - eps * oracle.logsumexp(L * LN2, axis=0)
        if self._bad(self.g):
            self.first_bad = min(self.first_bad, step)

    def check(self, which, measure, eps):
        fp = self.f[which]
        v = np.zeros(8)
        if measure:
            fn = self.f[1 - which]
            with np.errstate(over="ignore", invalid="ignore"):
                r = np.where(self.a > 0, self.a * np.exp((fp - fn) / eps), 0.0)
            v[0] = np.abs(r - self.a).sum()
            v[1] = r.sum()
        with np.errstate(invalid="ignore"):
            v[2] = np.where(self.a > 0, self.a * fp, 0.0).sum()
            v[3] = np.where(self.b > 0, self.b * self.g, 0.0).sum()
        v[4], v[5] = np.isnan(fp).sum(), np.isnan(self.g).sum()
        v[6], v[7] = (fp == np.inf).sum(), (self.g == np.inf).sum()
        return v

    def read_first_bad(self):
        return self.first_bad


def _problem(seed, n, m, d, nonuniform):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d))
    y = rng.standard_normal((m, d)) + 0.5
    if nonuniform:
        a = rng.uniform(0.5, 1.5, n)
        b = rng.uniform(0.5, 1.5, m)
        a[3] = 0.0
        b[5] = 0.0
        a, b = a / a.sum(), b / b.sum()
    else:
        a, b = np.full(n, 1.0 / n), np.full(m, 1.0 / m)
    eps = 0.05 * float(np.mean(((x[:, None, :] - y[None, :, :]) ** 2).sum(-1)))
    return x, y, a, b, eps


CASES = {
    # name: (seed, n, m, d, nonuniform, eps-scale, threshold, max_iters, schedule)
    "converges": (1, 97, 64, 3, False, 1.0, 1e-3, 400, None),
    "nonuniform": (2, 130, 77, 5, True, 1.0, 1e-6, 300, None),
    "fixed_iters": (3, 64, 50, 2, False, 1.0, 1e-300, 23, None),
    "annealed": (4, 80, 90, 3, False, 0.3, 1e-4, 500, (4.0, 0.7)),
}


def _run_shard(case, comm, world, rank):
    seed, n, m, d, nonu, es, thr, mi, sch = CASES[case]
    x, y, a, b, eps = _problem(seed, n, m, d, nonu)
    sched = EpsilonSchedule(eps * es, *(sch or ()))
    lo, hi = shard_rows(n, world, rank)
    eng = NumpyShardEngine(x[lo:hi], y, a[lo:hi], b)
    which, iters, conv, errs, duals = sharded_loop(eng, comm, sched, thr, mi, 10)
    return dict(f=eng.f[which], g=eng.g, iters=iters, conv=conv, errs=errs, duals=duals, lo=lo)


def _reference(case):
    seed, n, m, d, nonu, es, thr, mi, sch = CASES[case]
    x, y, a, b, eps = _problem(seed, n, m, d, nonu)
    sched = oracle.EpsilonScheduleOracle(eps * es, *(sch or ())) if sch else eps * es
    return oracle.sinkhorn(oracle.PointCloudOracle(x, y), a, b, sched, threshold=thr, max_iters=mi,
                           inner_iters=10)


def _compare(case, shards):
    ref = _reference(case)
    f = np.concatenate([s["f"] for s in sorted(shards, key=lambda s: s["lo"])])
    scale_f = np.max(np.abs(ref["f"][np.isfinite(ref["f"])]))
    fin = np.isfinite(ref["f"])
    assert np.array_equal(fin, np.isfinite(f))
    assert np.max(np.abs(f[fin] - ref["f"][fin])) <= 1e-10 * scale_f
    for s in shards:  # g replicated bitwise on every rank
        assert np.array_equal(s["g"], shards[0]["g"])
        assert s["iters"] == ref["iterations"] and s["conv"] == ref["converged"]
        np.testing.assert_allclose(s["errs"], ref["errors"], rtol=1e-6, atol=1e-14)
        np.testing.assert_allclose(s["duals"], ref["dual_trace"], rtol=1e-10)
    gfin = np.isfinite(ref["g"])
    assert np.max(np.abs(shards[0]["g"][gfin] - ref["g"][gfin])) <= 1e-10 * np.max(np.abs(ref["g"][gfin]))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _gloo_worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, _run_shard(case, TorchComm(), world, rank)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["converges", "nonuniform", "fixed_iters", "annealed"])
def test_gloo_two_ranks_match_unsharded_oracle(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    shards = [q.get(timeout=300)[1] for _ in procs]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    _compare(case, shards)


@pytest.mark.parametrize("world", [1, 3])
def test_thread_ranks_match_unsharded_oracle(world):
    comms = ThreadComm.group(world)
    out = [None] * world

    def run(r):
        out[r] = _run_shard("nonuniform", comms[r], world, r)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    _compare("nonuniform", out)


def test_bad_potential_is_raised_on_every_rank_like_the_oracle():
    """A denormal eps overflows every (g - C)/eps to -inf, so f_1 = +inf.  The
    reference raises ValueError when the g half-step is fed that potential
    (geometry.py:65-72); every rank raises it, at the first check, for
    iteration 1 (solve.cu's step numbering)."""
    world = 2
    comms = ThreadComm.group(world)
    seen = [None] * world
    x, y, a, b, _ = _problem(7, 40, 30, 2, False)
    with pytest.raises(ValueError):
        with np.errstate(all="ignore"):
            oracle.sinkhorn(oracle.PointCloudOracle(x, y), a, b, 1e-310, threshold=1e-3,
                            max_iters=100, inner_iters=10)

    def run(r):
        lo, hi = shard_rows(40, world, r)
        eng = NumpyShardEngine(x[lo:hi], y, a[lo:hi], b)
        try:
            sharded_loop(eng, comms[r], EpsilonSchedule(1e-310), 1e-3, 100, 10)
        except ValueError as e:
            seen[r] = str(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert seen[0] is not None and seen[0] == seen[1]
    assert "iteration 1" in seen[0]


def test_nan_at_a_check_raises_diverged_on_every_rank():
    """NaN in g at a check iteration -> DivergedError(iteration=t) on all ranks
    (sinkhorn.py:176-180), decided from the rank-order-reduced check sums."""

    class NanAtThree(NumpyShardEngine):
        t = 0

        def cols_finalize(self, lall, eps, kappa_next, step):
            super().cols_finalize(lall, eps, kappa_next, step)
            if step == 2 * 3 + 1:
                self.g[0] = np.nan

    world = 2
    comms = ThreadComm.group(world)
    seen = [None] * world
    x, y, a, b, eps = _problem(8, 50, 40, 3, False)

    def run(r):
        lo, hi = shard_rows(50, world, r)
        eng = NanAtThree(x[lo:hi], y, a[lo:hi], b)
        try:
            sharded_loop(eng, comms[r], EpsilonSchedule(eps), 1e-300, 100, 3)
        except DivergedError as e:
            seen[r] = e.iteration

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert seen == [3, 3]


def test_shard_rows_partition():
    for n in (1, 7, 64, 65537):
        for w in (1, 2, 3, 8):
            if w > n:
                continue
            spans = [shard_rows(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


# ------------------------------------------------ peer-memory exchange protocol
def _gloo_exchange_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2201_12324_b200.sharded import p2p_exchange_supported
        comm = TorchComm()
        handles = comm.all_gather_bytes(bytes([rank]) * 64)   # IPC handles are 64 bytes
        objs = comm.all_gather_objects(("host", rank))
        q.put((rank, handles, objs, p2p_exchange_supported(comm)))
    finally:
        dist.destroy_process_group()


def test_gloo_exchange_handshake_host_logic():
    """The handle exchange of PeerExchange (64-byte CUDA IPC handles through the
    process group, in rank order) and the transport choice: gloo -> collective."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (h, o, s)) for r, h, o, s in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in range(2):
        handles, objs, supported = res[r]
        assert handles == [bytes([0]) * 64, bytes([1]) * 64]
        assert objs == [("host", 0), ("host", 1)]
        assert supported is False


def test_exchange_protocol_model_never_reads_a_stale_or_overwritten_slot():
    """Host model of csrc/p2p.cu's protocol (W ranks as threads with random
    delays): each epoch e every rank writes its tagged partial into slot
    (e & 1, rank) of every peer, then releases flag[rank] = e on every peer;
    the combine waits for all flags >= e and reads slot (e & 1).  Two slots
    must suffice: no rank may ever read a partial of the wrong epoch."""
    import random
    import threading as th
    W, E = 4, 200
    slots = [[[None] * W for _ in range(2)] for _ in range(W)]   # [owner][slot][writer]
    flags = [[0] * W for _ in range(W)]                             # [owner][writer]
    cv = th.Condition()
    errors = []

    def rank(r):
        rng = random.Random(r)
        for e in range(1, E + 1):
            for s in rng.sample(range(W), W):           # push in any order
                slots[s][e & 1][r] = (r, e)
                if rng.random() < 0.3:
                    th.Event().wait(0.0001)
            with cv:                                     # release after all stores
                for s in range(W):
                    flags[s][r] = e
                cv.notify_all()
            with cv:                                     # acquire: wait for every writer
                cv.wait_for(lambda: all(flags[r][w] >= e for w in range(W)))
            got = [slots[r][e & 1][w] for w in range(W)]
            if got != [(w, e) for w in range(W)]:
                errors.append((r, e, got))
            if rng.random() < 0.3:
                th.Event().wait(0.0002)

    ts = [th.Thread(target=rank, args=(r,)) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert not errors, errors[:3]


def test_device_counted_epoch_protocol_model():
    """Host model of the device-counted epochs of csrc/p2p.cu, which let the
    native sharded loop replay the same launches inside CUDA graphs: the push
    (finalize) and every block of the combine use E = done + 1 read from the
    rank's own buffer; each combine block takes a ticket after reading E and
    the last one sets done = E.  Blocks run as threads in any order (as if not
    co-resident); every 10th epoch a single-block check exchange with its own
    counter runs in the same stream order.  No block may see a wrong epoch,
    a stale slot, or a wrong rank-order total."""
    import random
    import threading as th
    W, E, B = 3, 120, 3
    slots = [[[None] * W for _ in range(2)] for _ in range(W)]   # [owner][slot][writer]
    flags = [[0] * W for _ in range(W)]
    chk_slots = [[[None] * W for _ in range(2)] for _ in range(W)]
    chk_flags = [[0] * W for _ in range(W)]
    done = [0] * W          # header EPOCH word per rank
    ticket = [0] * W        # header TICKET word per rank
    chk_done = [0] * W      # header CHK_EPOCH word per rank
    lock = th.Lock()
    cv = th.Condition()
    errors = []

    def combine_block(r, e_expected, rng):
        ep = done[r] + 1                                # exchange_epoch(local, 0)
        if ep != e_expected:
            errors.append(("epoch", r, ep, e_expected))
        if rng.random() < 0.5:
            th.Event().wait(0.0001)
        with cv:
            cv.wait_for(lambda: all(flags[r][w] >= ep for w in range(W)))
        got = [slots[r][ep & 1][w] for w in range(W)]
        if got != [(w, ep) for w in range(W)]:
            errors.append(("slot", r, ep, got))
        with lock:                                      # atomicAdd(ticket) == gridDim - 1
            ticket[r] += 1
            last = ticket[r] == B
            if last:
                ticket[r] = 0
        if last:
            done[r] = ep

    def rank(r):
        rng = random.Random(100 + r)
        for e in range(1, E + 1):
            ep = done[r] + 1                            # push kernel: same formula
            for s in rng.sample(range(W), W):
                slots[s][ep & 1][r] = (r, ep)
            with cv:
                for s in range(W):
                    flags[s][r] = ep
                cv.notify_all()
            blocks = [th.Thread(target=combine_block, args=(r, e, random.Random(e * 7 + r + b)))
                      for b in range(B)]
            for b in rng.sample(blocks, B):
                b.start()
            for b in blocks:                            # stream order: the combine completes
                b.join()
            if done[r] != e:
                errors.append(("done", r, done[r], e))
            if e % 10 == 0:                             # check exchange (one block)
                ce = chk_done[r] + 1
                for s in range(W):
                    chk_slots[s][ce & 1][r] = (r, ce, float(r + 1))
                with cv:
                    for s in range(W):
                        chk_flags[s][r] = ce
                    cv.notify_all()
                    cv.wait_for(lambda: all(chk_flags[r][w] >= ce for w in range(W)))
                vals = [chk_slots[r][ce & 1][w] for w in range(W)]
                if [v[:2] for v in vals] != [(w, ce) for w in range(W)]:
                    errors.append(("chk", r, ce, vals))
                tot = 0.0
                for w in range(W):                      # fixed rank order
                    tot += vals[w][2]
                if tot != W * (W + 1) / 2:
                    errors.append(("tot", r, tot))
                chk_done[r] = ce

    ts = [th.Thread(target=rank, args=(r,)) for r in range(W)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    assert not errors, errors[:3]
    assert done == [E] * W and chk_done == [E // 10] * W


def test_peer_timeout_on_one_rank_raises_on_every_rank():
    """A rank whose peer-memory wait timed out (status word != 0) must not leave
    the others blocked in the check's gather: its status travels with the
    check sums and EVERY rank raises at the same check."""

    class FakeP2P:
        def __init__(self, bad):
            self.bad = bad

        def status(self):
            return 1 if self.bad else 0

    class ExchangingEngine(NumpyShardEngine):
        comm = None

        def cols_exchange(self, p2p, kappa, eps, kappa_next, step):
            lall = self.comm.all_gather_rows(self.cols_partial(kappa))
            self.cols_finalize(lall, eps, kappa_next, step)

    world = 2
    comms = ThreadComm.group(world)
    seen = [None] * world
    x, y, a, b, eps = _problem(9, 44, 30, 3, False)

    def run(r):
        lo, hi = shard_rows(44, world, r)
        eng = ExchangingEngine(x[lo:hi], y, a[lo:hi], b)
        eng.comm = comms[r]
        try:
            sharded_loop(eng, comms[r], EpsilonSchedule(eps), 1e-300, 100, 10, p2p=FakeP2P(r == 1))
        except RuntimeError as e:
            seen[r] = str(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert all(not t.is_alive() for t in ts)
    assert seen[0] is not None and seen[0] == seen[1] and "timed out" in seen[0]
