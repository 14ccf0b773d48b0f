"""ZeRO-1 data-parallel step logic at world_size 2 over torch.distributed/gloo
on CPU -- the host-side algorithm session.cu runs with NCCL on the GPUs:

  * gradient exchange: every rank receives all ranks' bf16 chunks of its
    shard (shard_layout from the native library, src/comms.cpp:69-73) and sums
    them in ascending rank order in f32 (src/trainer.cpp:90-103);
  * global norm from per-shard 256-block partials + all-reduce;
  * AdamW on the shard with global-index RNG keys, then an all-gather of the
    padded bf16 slices (src/optim.cpp:112-176).

The result must equal the single-process reference trainer step bitwise."""
import os

import numpy as np
import pytest

from tests.helpers import bf16_grid_round, rng_floats

torch = pytest.importorskip("torch")

SIZES = {"embed": 1000, "layers.0.w_qkv": 3000, "final_g": 64, "lm_head": 777}


def _grads(rank):
    return {n: bf16_grid_round(rng_floats(100 + 7 * rank + i, s, -1, 1)) for i, (n, s) in enumerate(SIZES.items())}


def _params():
    return {n: bf16_grid_round(rng_floats(50 + i, s, -1, 1)) for i, (n, s) in enumerate(SIZES.items())}


def _worker(rank, world, port_num, out_q):
    import torch.distributed as dist
    from oracle import port
    from paper_2512_15306_b200 import session as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_num)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params = _params()
    mine = _grads(rank)
    ssq_local = 0.0
    shards = {}
    for n, size in SIZES.items():
        padded, pw = S.shard_layout(size, world)
        lo, hi = min(rank * pw, size), min((rank + 1) * pw, size)
        gpad = np.zeros(padded, np.float32)
        gpad[:size] = mine[n]
        allg = [torch.zeros(padded) for _ in range(world)]
        dist.all_gather(allg, torch.from_numpy(gpad))
        s = allg[0].numpy()[rank * pw:rank * pw + pw].copy()
        for w in range(1, world):
            s = (s + allg[w].numpy()[rank * pw:rank * pw + pw]).astype(np.float32)  # ascending, f32
        shards[n] = (s, lo, hi, pw, padded)
        if lo < hi:
            ssq_local += port.grad_norm_partials(s[:hi - lo])
    t = torch.tensor([ssq_local], dtype=torch.float64)
    dist.all_reduce(t)
    norm = float(np.sqrt(t.item()))
    scale = 0.5
    newp = {}
    for n, size in SIZES.items():
        s, lo, hi, pw, padded = shards[n]
        full_g = np.zeros(size, np.float32)
        full_g[lo:hi] = s[:hi - lo]
        z = np.zeros(size, np.float32)
        p_upd = port.adamw_tensor(n, params[n], z, z, full_g, seed=3, grad_scale=scale, lo=lo, hi=hi)[0] \
            if lo < hi else params[n]
        sl = np.zeros(pw, np.float32)
        sl[:hi - lo] = p_upd[lo:hi]
        parts = [torch.zeros(pw) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(sl))
        newp[n] = torch.cat(parts).numpy()[:size]
    out_q.put((rank, norm, {k: v.tobytes() for k, v in newp.items()}))
    dist.destroy_process_group()


def test_zero1_step_world2_matches_single_process():
    import socket
    import torch.multiprocessing as mp
    from oracle import port
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_num = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_num, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    # single-process reference: ascending-worker f32 sum, f64 block norm, unsharded AdamW
    g0, g1 = _grads(0), _grads(1)
    params = _params()
    ssq = 0.0
    want = {}
    for n in SIZES:
        g = (g0[n] + g1[n]).astype(np.float32)
        ssq += port.grad_norm_partials(g)
        z = np.zeros_like(g)
        want[n] = port.adamw_tensor(n, params[n], z, z, g, seed=3, grad_scale=0.5)[0]
    for rank, norm, newp in res:
        assert abs(norm - np.sqrt(ssq)) / np.sqrt(ssq) < 1e-12
        for n in SIZES:
            np.testing.assert_array_equal(np.frombuffer(newp[n], np.float32), want[n], err_msg=f"rank {rank} {n}")


# ---------------------------------------------------------------------------
# RunPlan::shard_weights: every rank holds only its ZeRO-1 slice of a block
# weight; the per-tensor absmax is the all-reduce MAX of the slice maxima, each
# rank casts its slice with that scale and the E4M3 codes are all-gathered
# (session.cu build_step_context).  Must equal the full-tensor cast bitwise.
# ---------------------------------------------------------------------------
WSIZES = {"layers.0.w_qkv": 3000, "layers.0.w_o": 1024, "layers.1.w_down": 777}


def _weights():
    return {n: bf16_grid_round(rng_floats(900 + i, s, -2, 2) * (1 + i)) for i, (n, s) in enumerate(WSIZES.items())}


def _worker_codes(rank, world, port_num, out_q):
    import torch.distributed as dist
    from oracle import port
    from paper_2512_15306_b200 import session as S
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_num)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    for n, w in _weights().items():
        padded, pw = S.shard_layout(w.size, world)
        lo, hi = min(rank * pw, w.size), min((rank + 1) * pw, w.size)
        local = port.absmax(w[lo:hi]) if lo < hi else 0.0
        t = torch.tensor([np.float32(local).view(np.int32)], dtype=torch.int32)  # |x| bit patterns order like floats
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        amax = float(np.int32(t.item()).view(np.float32))
        codes = np.zeros(pw, np.uint8)
        if lo < hi:
            codes[:hi - lo] = port.quantize_with_absmax(w[lo:hi], 0, amax)[0]
        parts = [torch.zeros(pw, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(codes))
        out[n] = (torch.cat(parts).numpy()[:w.size].tobytes(), port.absmax_scale(amax, 0))
    out_q.put((rank, out))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shard_weights_code_allgather_matches_full_cast(world):
    import socket
    import torch.multiprocessing as mp
    from oracle import port
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port_num = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker_codes, args=(r, world, port_num, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for n, w in _weights().items():
        amax = port.absmax(w)
        want_codes, want_scale = port.quantize_with_absmax(w, 0, amax)
        for rank, out in res:
            got, scale = out[n]
            np.testing.assert_array_equal(np.frombuffer(got, np.uint8), want_codes, err_msg=f"rank {rank} {n}")
            assert scale == want_scale
