"""Column sharding across ranks with world_size = 2 on CPU (gloo).

Each rank keeps rows [rank·N/G, (rank+1)·N/G) of every member (paper_2605_05819_b200.shard_rows),
computes its slice of every window with the float64 oracle, all-gathers the slices with gloo in the
[G][B][n_local] layout NCCL produces, and restores the canonical layout with the library's own gather
permutation (hc_unshard_host, the index map of the device kernel).  The sharded decode stack must equal
the unsharded oracle stack bit-for-bit (every output element is the same float64 dot product)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import linear
from oracle.packing import bf16_to_f64

D, KV, F, L, B = 128, 64, 256, 2, 3
GAINS = synth.STACK_GAINS


def _stack():
    layers, ranks = [], []
    for l in range(L):
        c = lambda n, k, s: synth.linear_case(900 + 10 * l + s, N=n, K=k, bits=4, r_stored=16, zeros="asym",
                                              unit_gain=GAINS[s])
        layers.append(dict(qkv=[c(D, D, 0), c(KV, D, 1), c(KV, D, 2)], o=[c(D, D, 3)],
                           upgate=[c(F, D, 4), c(F, D, 5)], down=[c(D, F, 6)]))
        ranks.append(dict(qkv=[16, 0, 8], o=[8], upgate=[16, 8], down=[16]))
    return layers, ranks


def _slice_case(case, lo, hi):
    out = dict(case)
    for k in ("codes", "scales", "zeros", "U"):
        out[k] = case[k][lo:hi]
    out["N"] = hi - lo
    return out


def _to_bits(a):
    return synth.f32_to_bf16_bits(linear.round_bf16(a).astype(np.float32))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2605_05819_b200 as hc
    layers, ranks = _stack()
    x = synth.activations(5, B, D)

    def window(members, rks, xin_bits, glue=False, resid=None):
        # local slices of every member -> [B][n_local] (bf16 bits), gather, unshard
        outs = []
        for m, r in zip(members, rks):
            lo, hi = hc.shard_rows(m["N"], world, rank)
            outs.append(linear.compensated_linear(_slice_case(m, lo, hi), r, x_bits=xin_bits))
        if glue:
            local = [linear.silu(outs[1]) * outs[0]]
            widths = [local[0].shape[1]]
        else:
            local, widths = outs, [o.shape[1] for o in outs]
        loc = np.concatenate(local, axis=1)
        if resid is not None:
            lo, hi = hc.shard_rows(resid.shape[1], world, rank)
            loc = loc + resid[:, lo:hi]
        loc_bits = _to_bits(loc)
        t = torch.from_numpy(loc_bits.astype(np.int32))               # gloo has no 16-bit integers
        gathered = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        g = torch.stack(gathered).numpy().astype(np.uint16)          # [G][B][n_local]
        return hc.unshard_host(g, world, B, widths)

    h = x
    for Lr, R in zip(layers, ranks):
        qkv = window(Lr["qkv"], R["qkv"], h)
        a = qkv[:, :D].copy()
        h1 = window(Lr["o"], R["o"], a, resid=bf16_to_f64(h))
        m = window(Lr["upgate"], R["upgate"], h1, glue=True)
        h = window(Lr["down"], R["down"], m, resid=bf16_to_f64(h1))
    ref = linear.stack_forward(layers, ranks, x)
    q.put((rank, bool(np.array_equal(bf16_to_f64(h), ref)), float(np.abs(bf16_to_f64(h) - ref).max())))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(300)
def test_column_sharded_stack_world2_equals_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, equal, err in res:
        assert equal, (rank, err)


def test_shard_rows_and_unshard_layout():
    import paper_2605_05819_b200 as hc
    assert hc.shard_rows(1024, 8, 3) == (384, 512)
    with pytest.raises(ValueError):
        hc.shard_rows(1024, 3, 0)
    with pytest.raises(ValueError):
        hc.shard_rows(128, 16, 0)                    # 8-row shards are below the 16-row block
    # G = 2, B = 2, two members of local widths (2, 1): gathered [G][B][3] -> [B][6]
    g = np.arange(2 * 2 * 3, dtype=np.uint16).reshape(2, 2, 3)
    out = hc.unshard_host(g, 2, 2, [2, 1])
    # member 0 full rows = rank0 (0,1) | rank1 (6,7); member 1 = rank0 (2) | rank1 (8)
    assert out[0].tolist() == [0, 1, 6, 7, 2, 8]
    assert out[1].tolist() == [3, 4, 9, 10, 5, 11]


def test_bench_spawns_one_rank_per_gpu():
    """bench.py --gpus N without WORLD_SIZE re-launches itself under torch.distributed.run with N ranks on
    127.0.0.1 (dry run: the command is printed, nothing runs); with WORLD_SIZE set (the driver's own
    torchrun launch) it does not re-spawn."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HC_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "4", "--steps", "5", "--warmup", "3"],
                         env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    cmd = json.loads(out.stdout.strip().splitlines()[-1])["spawn"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-6:] == ["--gpus", "4", "--steps", "5", "--warmup", "3"]
