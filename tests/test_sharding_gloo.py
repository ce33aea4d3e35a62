"""Multi-process (gloo, world_size 2) coverage of the N>1 paths on CPU.

* config 5: each rank computes its particle shard's statistics record, the
  records are exchanged with the same RecordExchange (all_gather_into_tensor)
  the NCCL path uses, and the fixed-order combine reproduces the unsharded
  update exactly (oracle restatement of the device record algebra);
* config 4: instance sharding covers every instance exactly once and ranks
  need no communication.
"""

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _config1_problem(n=96):
    sys.path.insert(0, str(ROOT))
    from oracle import mppi_oracle as O
    from paper_2104_13542_b200 import configs
    from paper_2104_13542_b200.kinematics import load_chain

    arm7 = load_chain("arm7.chain")
    kw = dict(configs.CONTROLLER_KW)
    kw.pop("seed")
    kw["particles"] = n
    oc = O.OracleController(arm7, configs.make_weights(1), configs.reach_goal_rotation(), configs.REACH_GOAL_POS,
                            True, **kw)
    # one full oracle step to get a non-trivial policy, then freeze the next iteration's inputs
    oc.step(configs.REACH_START, np.zeros(7))
    means, var = O.shifted(oc.means, oc.variances, 0.0, oc.sigma0_sq)
    eps = oc.eps_source()
    u = O.shape_controls(eps, means, var, oc.null)
    res = O.rollout_scores(configs.REACH_START, np.zeros(7), u, oc.dts, arm7, oc.weights, oc.goal_R, oc.goal_t,
                           True, oc.gamma, oc.tw)
    return O, oc, means, var, u, res["totals"]


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, str(ROOT))
        from paper_2104_13542_b200.sharded import RecordExchange, particle_shard

        O, oc, means, var, u, totals = _config1_problem()
        off, cnt = particle_shard(u.shape[0], world, rank)
        rec = O.shard_record(totals[off:off + cnt], u[off:off + cnt] - means[None], oc.beta)
        gathered = RecordExchange().all_gather(torch.from_numpy(rec)).numpy().reshape(world, -1)
        mu, v = O.combine_and_update(gathered, means, var, oc.alpha_mu, oc.alpha_sigma, oc.smin, oc.smax, oc.beta)
        out_q.put((rank, mu, v))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_particle_sharded_update_matches_unsharded(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    O, oc, means, var, u, totals = _config1_problem()
    w = O.weights_from_totals(totals, oc.beta)
    mu_ref, var_ref = O.blend_policy(means, var, u, w, oc.alpha_mu, oc.alpha_sigma, oc.smin, oc.smax)
    results.sort(key=lambda r: r[0])
    for _, mu, v in results:
        np.testing.assert_allclose(mu, mu_ref, atol=1e-12)
        np.testing.assert_allclose(v, var_ref, atol=1e-12)
    # every rank ends with the identical policy (no broadcast needed)
    np.testing.assert_array_equal(results[0][1], results[1][1])


def test_shard_arithmetic():
    sys.path.insert(0, str(ROOT))
    from paper_2104_13542_b200.batched import shard_instances
    from paper_2104_13542_b200.sharded import particle_shard

    for total in (1, 7, 500, 4096, 262144):
        for world in (1, 2, 3, 4, 8):
            if total < world:
                continue
            seen = []
            for r in range(world):
                a, b = shard_instances(total, world, r)
                seen.extend(range(a, b))
                off, cnt = particle_shard(total, world, r)
                assert (off, off + cnt) == (a, b)
            assert seen == list(range(total))


class _FakePeerOps:
    """Stand-in for the plan's IPC surface: rank r's buffers are the integers
    r*100 + {1, 2}; a handle is the pointer's text; opening maps it into this
    process as 10**6 + pointer."""

    def __init__(self, rank):
        self.rank = rank
        self.calls = []

    def peer_buffers(self, world):
        self.calls.append(("peer_buffers", world))
        return self.rank * 100 + 1, self.rank * 100 + 2

    def ipc_handle(self, ptr):
        return str(ptr).encode().ljust(64, b"\0")

    def ipc_open(self, handle):
        return 10 ** 6 + int(handle.rstrip(b"\0"))

    def ipc_close(self, ptr):
        self.calls.append(("close", ptr))

    def set_peers(self, rank, recv, flags):
        self.calls.append(("set_peers", rank, list(recv), list(flags)))


def _peer_worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, str(ROOT))
        from paper_2104_13542_b200.sharded import PeerExchange

        ops = _FakePeerOps(rank)
        ex = PeerExchange()
        tables = ex.attach(ops)
        ex.close(ops)
        out_q.put((rank, tables, ops.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_tables(world):
    """PeerExchange wiring over gloo: slot k of every rank's table addresses
    rank k's buffers — its own raw pointers in slot [rank], the opened IPC
    mappings elsewhere — and every opened mapping is closed again."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (recv, flags), calls in results:
        assert calls[0] == ("peer_buffers", world)
        for k in range(world):
            base = 0 if k == rank else 10 ** 6
            assert recv[k] == base + k * 100 + 1 and flags[k] == base + k * 100 + 2
        sp = [c for c in calls if c[0] == "set_peers"]
        assert sp == [("set_peers", rank, recv, flags)]
        closed = sorted(c[1] for c in calls if c[0] == "close")
        assert closed == sorted(x for k in range(world) if k != rank for x in (recv[k], flags[k]))


def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` without torchrun's environment re-executes
    itself under torch.distributed.run: the dry run
    (gloo, no GPU) must report two ranks and the N>1 default workload."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--dry-run"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(next(ln for ln in r.stdout.splitlines() if ln.startswith("{")))
    assert line["n_gpus"] == 2 and line["max_rank_seen"] == 1
    assert line["workload"] == "c4" and line["config"]["parallelism"] == "instance-sharded x2"
    # one GPU: unchanged default (the config-2 latency headline)
    r1 = subprocess.run([sys.executable, str(root / "bench.py"), "--dry-run"], cwd=root, env=env,
                        capture_output=True, text=True, timeout=120)
    line1 = json.loads(next(ln for ln in r1.stdout.splitlines() if ln.startswith("{")))
    assert line1["n_gpus"] == 1 and line1["workload"] == "c2"
    # a mismatched WORLD_SIZE fails loudly instead of running one GPU silently
    bad = dict(env, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r2 = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "8", "--dry-run"], cwd=root, env=bad,
                        capture_output=True, text=True, timeout=120)
    assert r2.returncode == 2
