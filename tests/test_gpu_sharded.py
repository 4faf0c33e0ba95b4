"""Row-sharded solver on the GPU, one B200.

* world 1 over a real NCCL process group: the sharded path (shard partial ->
  all_gather -> rank-order combine) must be BITWISE identical to the
  single-GPU solver, whose combine sees the same partials in the same order.
* W = 2, 3 ranks emulated by threads sharing the GPU (ThreadComm: every
  exchange goes through the host; no kernel waits on another rank): f (all
  shards), g, iterations and converged flag against the float64 oracle, and
  the regularised cost through reg_ot_cost_sharded.
"""

import os
import socket
import threading

import numpy as np
import pytest

import oracle
from paper_2201_12324_b200 import workloads

pytestmark = pytest.mark.gpu

POT_TOL = 1e-4
COST_TOL = 1e-5


@pytest.fixture(scope="module")
def otk():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_12324_b200 as m
    from paper_2201_12324_b200 import _native
    _native.lib()
    return m


def _rel(got, want):
    fin = np.isfinite(want)
    return np.max(np.abs(got[fin] - want[fin])) / np.max(np.abs(want[fin]))


@pytest.fixture(scope="module")
def nccl_world1():
    import torch
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("d,gen", [(3, "cfg1"), (64, "cfg2"), (128, "cfg4")])
def test_world1_nccl_is_bitwise_the_single_gpu_solver(otk, nccl_world1, d, gen):
    from paper_2201_12324_b200.sharded import solve_sinkhorn_sharded
    kw = dict(n=640, m=512) if gen != "cfg2" else dict(n=640, m=512, d=d)
    wl = getattr(workloads, gen)(**kw)
    from paper_2201_12324_b200 import _native as N
    geom = otk.PointCloudGeometry(wl.x, wl.y)
    geom.impl_flags = N.OTK_IMPL_NOPERSIST  # the launch-per-half-step loop the shards run
    single = otk.solve_sinkhorn(otk.LinearProblem(geom, wl.a, wl.b), wl.eps,
                                threshold=wl.threshold, max_iters=60)
    sh = solve_sinkhorn_sharded(wl.x, wl.y, wl.eps, wl.a, wl.b, threshold=wl.threshold,
                                max_iters=60)
    assert sh.iterations == single.iterations and sh.converged == single.converged
    assert np.array_equal(sh.f_local, single.f)
    assert np.array_equal(sh.g, single.g)
    np.testing.assert_array_equal(sh.errors, single.errors)


def _thread_solve(otk, wl, world, **kw):
    from paper_2201_12324_b200.sharded import ThreadComm, solve_sinkhorn_sharded, reg_ot_cost_sharded
    from paper_2201_12324_b200.sharded import shard_rows
    comms = ThreadComm.group(world)
    outs, costs, errs = [None] * world, [None] * world, []
    n = wl.shape[0]
    a = wl.a if wl.a is not None else np.full(n, 1.0 / n)
    b = wl.b if wl.b is not None else np.full(wl.shape[1], 1.0 / wl.shape[1])

    def run(r):
        try:
            o = solve_sinkhorn_sharded(wl.x, wl.y, wl.eps, wl.a, wl.b, comm=comms[r],
                                       gather_f=True, **kw)
            lo, hi = shard_rows(n, world, r)
            costs[r] = reg_ot_cost_sharded(o, wl.x[lo:hi], wl.y, a[lo:hi], b, comm=comms[r])
            outs[r] = o
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            comms[r].shared.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(600)
    if errs:
        raise errs[0]
    return outs, costs, a, b


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("gen,kw", [("cfg1", dict(n=600, m=520)),
                                    ("cfg2", dict(n=700, m=384, d=64)),
                                    ("cfg4", dict(n=900, m=450))])
def test_thread_ranks_match_oracle(otk, world, gen, kw):
    wl = getattr(workloads, gen)(**kw)
    # one check, at t = 20 (an fp32 fixed point can reach err == 0 <= 1e-300)
    outs, costs, a, b = _thread_solve(otk, wl, world, threshold=1e-300, max_iters=20,
                                      inner_iters=20)
    geom64 = oracle.PointCloudOracle(wl.x.astype(np.float64), wl.y.astype(np.float64))
    ref = oracle.sinkhorn(geom64, a, b, wl.eps, threshold=1e-300, max_iters=20)
    for o in outs:
        assert np.array_equal(o.g, outs[0].g)          # replicated bitwise
        assert np.array_equal(o.f, outs[0].f)
        assert o.iterations == 20
    assert _rel(outs[0].f, ref["f"]) <= POT_TOL
    assert _rel(outs[0].g, ref["g"]) <= POT_TOL
    tc, dual = oracle.reg_ot_cost(geom64, ref["f"], ref["g"], a, b, wl.eps)
    for c in costs:
        assert abs(c.transport_cost - tc) <= COST_TOL * abs(tc)
        assert abs(c.dual_objective - dual) <= COST_TOL * abs(dual)


def test_thread_ranks_converge_like_the_reference(otk):
    """Tolerance run: same iteration count / converged flag as the oracle."""
    wl = workloads.cfg1(n=512, m=512)
    outs, _, a, b = _thread_solve(otk, wl, 2, threshold=wl.threshold, max_iters=wl.max_iters)
    geom64 = oracle.PointCloudOracle(wl.x.astype(np.float64), wl.y.astype(np.float64))
    ref = oracle.sinkhorn(geom64, a, b, wl.eps, threshold=wl.threshold, max_iters=wl.max_iters)
    assert outs[0].iterations == ref["iterations"] and outs[0].converged == ref["converged"]
    assert len(outs[0].errors) == len(ref["errors"])


@pytest.mark.parametrize("d,gen", [(3, "cfg1"), (64, "cfg2")])
def test_world1_peer_exchange_is_bitwise_the_collective(otk, nccl_world1, d, gen):
    """The g half-step pushed over peer memory by its own last kernel (csrc/p2p.cu)
    gives the same bits as the NCCL all-gather + combine path (world 1: the
    rank is its own peer; no kernel waits on another process)."""
    from paper_2201_12324_b200.sharded import ShardedProblem
    kw = dict(n=700, m=515) if gen != "cfg2" else dict(n=700, m=515, d=d)
    wl = getattr(workloads, gen)(**kw)
    p2p = ShardedProblem(wl.x, wl.y, wl.a, wl.b, exchange="p2p")
    col = ShardedProblem(wl.x, wl.y, wl.a, wl.b, exchange="collective")
    assert p2p.exchange == "p2p" and col.exchange == "collective"
    for thr, its in ((wl.threshold, 60), (1e-300, 23)):
        a = p2p.solve(wl.eps, threshold=thr, max_iters=its)
        b = col.solve(wl.eps, threshold=thr, max_iters=its)
        assert a.iterations == b.iterations and a.converged == b.converged
        assert np.array_equal(a.f_local, b.f_local)
        assert np.array_equal(a.g, b.g)
        np.testing.assert_array_equal(a.errors, b.errors)
    assert p2p.p2p.status() == 0
    assert p2p.loop == "native" and col.loop == "python"


@pytest.mark.parametrize("d,gen", [(3, "cfg1"), (64, "cfg2"), (128, "cfg4")])
def test_world1_native_sharded_loop_matches_python_loop_and_single_gpu(otk, nccl_world1, d, gen,
                                                                       monkeypatch):
    """otk_solve_pointcloud_sharded (C++ loop, graph-captured check periods,
    device-counted exchange epochs, check sums exchanged on the device) vs the
    Python loop over the same peer exchange and vs the single-GPU general loop:
    bitwise equal f, g, errors, dual trace, iterations -- over repeated solves
    (the epoch sequence continues across solves and across the two loops)."""
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200.sharded import ShardedProblem
    kw = dict(n=700, m=515) if gen != "cfg2" else dict(n=700, m=515, d=d)
    wl = getattr(workloads, gen)(**kw)
    sp = ShardedProblem(wl.x, wl.y, wl.a, wl.b, exchange="p2p")
    assert sp.loop == "native"
    geom = otk.PointCloudGeometry(wl.x, wl.y)
    geom.impl_flags = N.OTK_IMPL_NOPERSIST
    prob = otk.LinearProblem(geom, wl.a, wl.b)
    for rep in range(2):
        for thr, its in ((wl.threshold, 60), (1e-300, 23), (1e-300, 41)):
            single = otk.solve_sinkhorn(prob, wl.eps, threshold=thr, max_iters=its)
            sp.loop = "native"
            nat = sp.solve(wl.eps, threshold=thr, max_iters=its)
            sp.loop = "python"
            py = sp.solve(wl.eps, threshold=thr, max_iters=its)
            for o in (nat, py):
                assert o.iterations == single.iterations and o.converged == single.converged
                assert np.array_equal(o.f_local, single.f) and np.array_equal(o.g, single.g)
                np.testing.assert_array_equal(o.errors, single.errors)
                np.testing.assert_array_equal(o.dual_trace, single.dual_trace)
    sp.loop = "native"
    assert sp.p2p.status() == 0
    sp.solve(wl.eps, threshold=1e-300, max_iters=30)
    assert sp.launches_last > 0


def test_world1_native_sharded_loop_failure_paths(otk, nccl_world1):
    """Same exceptions at the same iteration as the single-GPU solver: a warm
    start with NaN (ValueError, geometry.py:65-72) and divergence
    (DivergedError, sinkhorn.py:176-180)."""
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200.sharded import ShardedProblem
    wl = workloads.cfg2(n=600, m=400, d=64)
    sp = ShardedProblem(wl.x, wl.y, exchange="p2p")
    geom = otk.PointCloudGeometry(wl.x, wl.y)
    geom.impl_flags = N.OTK_IMPL_NOPERSIST
    prob = otk.LinearProblem(geom)
    g0 = np.zeros(400)
    g0[5] = np.nan
    for call in (lambda: sp.solve(wl.eps, g_init=g0), lambda: otk.solve_sinkhorn(prob, wl.eps, g_init=g0)):
        with pytest.raises(ValueError):
            call()
    outcomes = []
    for call in (lambda: sp.solve(1e-30, inner_iters=1, max_iters=20),
                 lambda: otk.solve_sinkhorn(prob, 1e-30, inner_iters=1, max_iters=20)):
        try:
            o = call()
            outcomes.append(("ok", o.iterations))
        except otk.DivergedError as e:
            outcomes.append(("diverged", e.iteration))
        except ValueError as e:
            outcomes.append(("value", str(e)))
    assert outcomes[0] == outcomes[1], outcomes
    # the exchange is still consistent after the failures
    a = sp.solve(wl.eps, threshold=1e-300, max_iters=12)
    b = otk.solve_sinkhorn(prob, wl.eps, threshold=1e-300, max_iters=12)
    assert np.array_equal(a.g, b.g)


def test_peer_exchange_wait_times_out_instead_of_hanging(otk, nccl_world1):
    """A combine whose peers never signal (epoch far ahead) gives up after its
    timeout, reports it through the status word and yields NaN, not a hang."""
    import torch
    from paper_2201_12324_b200 import _native as N
    from paper_2201_12324_b200._device import stream
    from paper_2201_12324_b200.sharded import PeerExchange, TorchComm
    m = 300
    px = PeerExchange(TorchComm(), m)
    out = torch.empty(m, dtype=torch.float32, device="cuda")
    base = torch.zeros(m, dtype=torch.float32, device="cuda")
    N.check(N.lib().otk_exchange_finalize(px.local, 1, m, 1000, N.ptr(base), N.OTK_FIN_SOLVER, 1.0,
                                          1.0, N.ptr(out), None, None, 0, 50, stream()))
    torch.cuda.synchronize()
    assert px.status() == 1
    assert torch.isnan(out).all()
    px.close()
