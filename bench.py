"""FP8 training throughput (tokens/s + MFU) of the LLMQ training step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config qwen2.5-0.5b] [--micro-batch B]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N ...
    python bench.py --impl reference ...      # the reference CPU implementation (oracle/_ref)

One step = one full trainer step (src/trainer.cpp:64-110): weight FP8 quantization
(build_step_context), forward + backward of one micro-batch per rank with
GradAccumulator SR, (ZeRO-1 gradient exchange when N > 1), global grad norm, clip,
AdamW and (N > 1) the bf16 parameter all-gather.  Synthetic uniform token ids,
random-init weights of the named shape (no network, no checkpoints).
Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

TOKENS_PER_OPT_STEP = 500_000

# B200 dense spec peaks used by the reference's MFU formula (src/memplan.cpp:307-312)
P_FP8_SPEC = 4.5e15
P_BF16_SPEC = 2.25e15


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", str(self.idx)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref): bounded samples of the same workload
# ---------------------------------------------------------------------------
def _ref_sample_seconds(cfg7_full, layers: int, tokens_per_seq: int, seed: int) -> float:
    from oracle import ref as R
    import numpy as np
    cfg7 = list(cfg7_full)
    cfg7[0] = layers
    m = R.RefModel(cfg7, seed, grad_e5m2=True)
    toks = np.random.default_rng(seed).integers(0, cfg7[5], size=tokens_per_seq + 1, dtype=np.int32)
    return m.time_step(toks, 1, 0)


def _ref_warm(_i):
    from oracle import ref as R
    return R.available()


def _ref_worker(args):
    cfg7, layers, tps, seed = args
    return _ref_sample_seconds(cfg7, layers, tps, seed)


def cpu_reference_model(cfg, sample_tokens: int) -> dict:
    """Per-token cost model of the reference step (src/trainer.cpp:64-110) for the
    full model, from samples at the real widths (one block
    fwd+bwd at the real d/F/H with T_cpu = 128 tokens, plus the CE at the real
    vocabulary, scaled by layers and tokens and labelled extrapolated):
      per-layer cost = t(2 layers) - t(1 layer), both with a 1024-id vocabulary
        (the embedding/CE share cancels), sample_tokens tokens in one sequence;
      the rest (embedding, final norm, LM head + CE at the real vocabulary) =
        t(1 layer, real V, ce_tokens) - per-layer cost at ce_tokens, scaled to
        sample_tokens (linear in tokens)."""
    cfg7 = cfg.as_list()
    small = list(cfg7)
    small[5] = 1024
    t1 = _ref_sample_seconds(small, 1, sample_tokens, 1)
    t2 = _ref_sample_seconds(small, 2, sample_tokens, 2)
    per_layer = max(t2 - t1, 1e-9)
    ce_tokens = min(sample_tokens, 16)
    tce = _ref_sample_seconds(cfg7, 1, ce_tokens, 3)
    # the attention term of per_layer grows with context; at ce_tokens the layer costs ~ linear share
    rest = max(tce - per_layer * ce_tokens / sample_tokens, 0.0) * sample_tokens / ce_tokens
    t_full = rest + cfg.n_layers * per_layer  # seconds per sample_tokens tokens, one core
    return {"t1": t1, "t2": t2, "t_ce": tce, "ce_tokens": ce_tokens, "t_full": t_full,
            "rate_1core": sample_tokens / t_full}


def cpu_reference_rate(cfg, sample_tokens: int, cores: int, model: dict | None = None, pool=None) -> dict:
    """tokens/s of the reference step on `cores` host cores: the one-core rate of
    the cost model, times the measured parallel efficiency of `cores`
    independent reference processes each running the one-layer, 1024-id-vocabulary
    sample of the cost model (`pool`:
    an already-started process pool, reused across steps so a step times the
    samples and not interpreter start-up)."""
    import multiprocessing as mp
    m = model or cpu_reference_model(cfg, sample_tokens)
    rate, wall = m["rate_1core"], 0.0
    if cores > 1:
        cfg7 = cfg.as_list()
        cfg7[5] = 1024  # the t1 sample (1 layer, 1024-id vocabulary): ~5 s per process
        own = pool is None
        if own:
            pool = mp.get_context("spawn").Pool(cores)
        try:
            t0 = time.perf_counter()
            ts = pool.map(_ref_worker, [(cfg7, 1, sample_tokens, 10 + i) for i in range(cores)], chunksize=1)
            wall = time.perf_counter() - t0
        finally:
            if own:
                pool.close()
                pool.join()
        rate = m["rate_1core"] * cores * min(1.0, (sum(ts) / max(wall, 1e-9)) / cores)
    return {"value": rate, "rate_1core": m["rate_1core"], "t_sample_1layer_s": m["t1"], "t_sample_2layer_s": m["t2"],
            "sample_tokens": sample_tokens, "wall_s": wall}


def _sample_text(cfg, sample_tokens, m) -> str:
    return (f"unmodified reference train step (src/trainer.cpp:64-110, oracle/_ref): per-layer cost from 1- and "
            f"2-layer samples at the real widths with {sample_tokens} tokens (t1={m['t1']:.2f}s t2={m['t2']:.2f}s, "
            f"1024-id vocab), embedding + LM head + CE at the real vocab from a {m['ce_tokens']}-token sample "
            f"(t={m['t_ce']:.2f}s); extrapolated to {cfg.n_layers} layers, linear in tokens (attention context "
            f"{sample_tokens} instead of {cfg.seq_len})")


def fp8_gemm_bytes_per_step(cfg, M: int) -> float:
    """Algorithmic HBM bytes of the block FP8 GEMMs of one step (operands read once,
    outputs written once): per layer 4 forward (E4M3 x E4M3 -> bf16, the down-proj also
    reads the residual), 4 dgrad (grad codes x weight codes -> bf16) and 4 wgrad
    (grad codes x activation codes -> SR read-modify-write of the bf16 accumulator)."""
    d, F = cfg.d_model, cfg.d_ff
    q, Hh = cfg.qkv_dim(), F // 2
    per_layer = 0.0
    for n_out, k_in in ((q, d), (d, d), (F, d), (d, Hh)):  # linear (out, in)
        per_layer += M * k_in + n_out * k_in + 2 * M * n_out        # forward
        per_layer += M * n_out + n_out * k_in + 2 * M * k_in        # dgrad
        per_layer += M * n_out + M * k_in + 4 * n_out * k_in        # wgrad (+ accumulator RMW)
    per_layer += 2 * M * d                                          # down-proj residual read
    return per_layer * cfg.n_layers


def run_reference_arm(args, cfg, B, T, world):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libqtrain_ref.so not built"}))
        return
    cores = os.cpu_count() or 1
    sample_tokens = args.ref_sample_tokens
    model = cpu_reference_model(cfg, sample_tokens)  # warm-up + the per-layer cost model
    import multiprocessing as mp
    with mp.get_context("spawn").Pool(cores) as pool:
        # start every worker and load the reference library once, outside the timed steps
        pool.map(_ref_warm, range(cores), chunksize=1)
        times = [cpu_reference_rate(cfg, sample_tokens, cores, model, pool)["value"] for _ in range(args.steps)]
    value = statistics.median(times)
    fp8_f, bf16_f = cfg.flops_per_token()
    line = {
        "impl": "reference", "metric": "fp8_train_tokens_per_sec", "value": value, "unit": "tokens/s",
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp8(e4m3 fwd / e5m2 grads) emulated on CPU", "data": "synthetic",
        "config": {"workload": args.config, "model": args.config, "global_batch": args.grad_accum * B * max(world, 1),
                   "micro_batch": B, "grad_accum": args.grad_accum, "seq_len": T, "parallelism": "cpu processes"},
        "mfu": value * (fp8_f / P_FP8_SPEC + bf16_f / P_BF16_SPEC),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "reference",
                         "sample": _sample_text(cfg, sample_tokens, model) + f"; each step = {cores} independent "
                                                                                     f"reference processes"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="qwen2.5-0.5b")
    ap.add_argument("--micro-batch", type=int, default=0)
    ap.add_argument("--grad-accum", type=int, default=0,
                    help="micro-batches per optimizer step (RunPlan::ga_steps); a step = one optimizer step. "
                         "0 = the paper's protocol: ~500k tokens per optimizer step per GPU (PAPER.md:366)")
    ap.add_argument("--seq", type=int, default=0)
    ap.add_argument("--grads", default="e5m2", choices=["e4m3", "e5m2"])
    ap.add_argument("--recompute", default="")
    ap.add_argument("--moments", default="f32", choices=["f32", "bf16_sr"])
    ap.add_argument("--shard-grads", action="store_true")
    ap.add_argument("--shard-weights", action="store_true")
    ap.add_argument("--offload", default="", help="RunPlan::offload categories: x,m,v,master,weights,grads")
    ap.add_argument("--transfer-policy", default="double_buffer", choices=["zero_copy", "double_buffer"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample-tokens", type=int, default=128)
    ap.add_argument("--profile-json", default="")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    from paper_2512_15306_b200 import session as S
    cfg = S.PRESETS[args.config]
    # micro-batch per GPU: the paper picks the fastest that fits; 7B at 12
    # (148 GB) runs 2.6 % faster than at 8 under the same accumulation (scripts/gpu_mb7b.sh)
    default_mb = {"tiny": 4, "qwen2.5-0.5b": 16, "qwen2.5-1.5b": 8, "llama-7b": 12, "qwen2.5-14b": 4}
    B = args.micro_batch or default_mb.get(args.config, 8)
    T = args.seq or cfg.seq_len
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.grad_accum <= 0:
        # the reference's throughput table is measured at a 500k-token optimizer batch
        # ("trained at a per-step batch size of 500k"); per GPU, so the
        # per-rank work stays fixed as N grows (weak scaling)
        args.grad_accum = max(1, round(TOKENS_PER_OPT_STEP / (B * T)))
    if args.impl == "reference":
        run_reference_arm(args, cfg, B, T, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [S.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    GA = max(1, args.grad_accum)
    plan = S.RunPlan(micro_batch=B, ga_steps=GA, recompute=tuple(x for x in args.recompute.split(",") if x),
                     moments=args.moments, shard_grads=args.shard_grads, shard_weights=args.shard_weights,
                     offload=tuple(x for x in args.offload.split(",") if x), transfer_policy=args.transfer_policy)
    sess = S.Session(cfg, S.PrecisionMap(backward_grads=args.grads), plan, S.AdamWHyper(), seed=1234, rank=rank,
                     world=world, nccl_id=nccl_id, device=local)
    sess.init_params(1234)
    stream = torch.cuda.ExternalStream(sess.stream)

    # synthetic uniform token ids (tests/test_model.cpp:29-35 layout: B*(T+1) per micro-batch)
    nbatches = 4
    g = np.random.default_rng(1000 + rank)
    host = [g.integers(0, cfg.vocab, size=GA * B * (T + 1), dtype=np.int32) for _ in range(nbatches)]
    dev = [torch.from_numpy(h).cuda() for h in host]
    pinned = [torch.from_numpy(h).pin_memory() for h in host]

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    # ---- warmup (also first-launch attribute setup)
    for i in range(args.warmup):
        sess.train_step(dev[i % nbatches], B, step=i, sync=False)
    sess.sync()
    try:
        kernels, other_nodes = sess.count_step_kernels(dev[0], B)  # exact: the step captured, not run
        launch_basis = "kernel nodes of the step captured into a CUDA graph"
    except Exception as e:  # a transport that cannot be captured (multi-rank): count in the profiled step
        kernels, other_nodes = None, None
        launch_basis = f"capture unavailable ({type(e).__name__}); launches of the profiled step"

    # ---- timed region: inputs resident in HBM; activations (GBs) >> 126 MB L2
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for i in range(args.steps):
        sess.train_step(dev[i % nbatches], B, step=args.warmup + i, sync=False)
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()

    # ---- end to end through the public API: pinned host tokens H2D + loss D2H every step
    h2d = GA * B * (T + 1) * 4
    d2h = 4 + 4
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    losses = []
    for i in range(args.steps):
        loss, norm = sess.train_step(pinned[i % nbatches].numpy(), B, step=args.warmup + args.steps + i, sync=True)
        losses.append(loss)
    e1.record(stream)
    e1.synchronize()
    barrier()
    ms_e2e = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = t.item()

    # ---- per-kernel-class roofline pass (CUDA events around every launch, one step)
    sess.set_profile(True)
    sess.train_step(dev[0], B, step=10_000, sync=True)
    prof = sess.profile()
    sess.set_profile(False)
    if kernels is None:
        kernels = int(sum(v["launches"] for v in prof.values()))

    tokens_per_step = GA * B * T * world
    value = tokens_per_step / (ms / 1e3)
    e2e_value = tokens_per_step / (ms_e2e / 1e3)
    fp8_f, bf16_f = cfg.flops_per_token()
    mfu = value / world * (fp8_f / P_FP8_SPEC + bf16_f / P_BF16_SPEC)
    peaks = _peaks()
    # dominant kernel class = largest device-time share of the profiled step
    total_ms = sum(v["ms"] for v in prof.values())
    dom_name, dom = max(prof.items(), key=lambda kv: kv[1]["ms"])
    if dom_name.startswith(("gemm", "attn")):
        achieved = dom["work"] / (dom["ms"] / 1e3) / 1e12
        mult = 2.0 if dom_name == "gemm_fp8" else 1.0  # attention / LM head: bf16
        # the kernels are timed inside a long step: the sustained rate is the denominator
        peak = peaks["bf16_tflops_sustained"] * mult
        roof = {"kernel": dom_name, "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak,
                "peak_basis": (f"2 x measured bf16 sustained (FP8 dense rate = 2x BF16 on sm_100)"
                               if dom_name == "gemm_fp8" else "measured bf16 sustained") + f" [{peaks['src']}]",
                "peak_burst": peaks["bf16_tflops"] * mult, "frac_burst": achieved / (peaks["bf16_tflops"] * mult),
                "launches": dom["launches"], "share_of_step": dom["ms"] / total_ms, "traffic": None,
                "algorithmic_flops_per_launch": dom["work"] / max(dom["launches"], 1)}
        fp8p = ROOT / "profiles" / "fp8_gemm_peak.json"
        if dom_name == "gemm_fp8" and fp8p.exists():
            try:
                fp = json.loads(fp8p.read_text())
                roof["peak_fp8_gemm_measured"] = fp["tflops"]
                roof["frac_vs_fp8_gemm_measured"] = achieved / fp["tflops"]
                roof["peak_fp8_gemm_measured_basis"] = fp["how"]
            except Exception:
                pass
    else:
        achieved = dom["work"] / (dom["ms"] / 1e3) / 1e9
        roof = {"kernel": dom_name, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "peak_basis": f"measured copy [{peaks['src']}]",
                "launches": dom["launches"], "share_of_step": dom["ms"] / total_ms, "traffic": None}
    if dom_name == "gemm_fp8":
        roof["algorithmic_bytes_per_launch"] = GA * fp8_gemm_bytes_per_step(cfg, B * T) / max(dom["launches"], 1)
    # DRAM bytes per launch of the dominant class from the committed ncu capture of one step
    # (scripts/traffic_summary.py; cold-cache serialised replay), when it matches this config
    tf = next((ROOT / "profiles" / f"r{r:02d}_traffic_0.5b.json" for r in (2, 1)
               if (ROOT / "profiles" / f"r{r:02d}_traffic_0.5b.json").exists()), ROOT / "profiles" / "r01_traffic_0.5b.json")
    if args.config == "qwen2.5-0.5b" and B == 16 and tf.exists():
        try:
            t = json.loads(tf.read_text())["classes"].get(dom_name)
            if t:
                # the capture is one GA = 1 step; the profiled step here has GA micro-steps
                per_call = t["dram_bytes_per_launch"] * t["launches"] * GA / max(dom["launches"], 1)
                roof["traffic"] = per_call
                roof["traffic_unit"] = "bytes/launch (dram read+write, ncu)"
                roof["traffic_source"] = str(tf.relative_to(ROOT))
        except Exception:
            pass
    classes = {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                   ("tflops" if k.startswith(("gemm", "attn")) else "gbs"):
                       round(v["work"] / (v["ms"] / 1e3) / (1e12 if k.startswith(("gemm", "attn")) else 1e9), 1)}
               for k, v in prof.items()}

    line = {
        "metric": "fp8_train_tokens_per_sec", "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp8", "data": "synthetic",
        "config": {"workload": args.config, "model": args.config, "global_batch": GA * B * world, "micro_batch": B,
                   "grad_accum": GA, "tokens_per_step": GA * B * T * world, "seq_len": T, "parallelism": f"dp{world}" + ("+zero1" if world > 1 else ""),
                   "grads": args.grads, "recompute": args.recompute or "none", "moments": args.moments,
                   "shard_grads": args.shard_grads, "shard_weights": args.shard_weights,
                   "offload": args.offload or "none", "transfer_policy": args.transfer_policy,
                   "l2": "activations/logits (GBs) exceed the 126 MB L2; no explicit flush"},
        "mfu": mfu,
        "mfu_basis": "reference formula (src/memplan.cpp:264-312) vs B200 dense spec 4.5 PF fp8 / 2.25 PF bf16",
        "roofline": roof,
        "kernel_classes": classes,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": kernels * args.steps,
        "gpu_launches_per_step": kernels,
        "gpu_launches_basis": launch_basis,
        "clocks": clk,
        "loss_last": losses[-1] if losses else None,
        "device_bytes": sess.device_bytes,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            m = cpu_reference_model(cfg, args.ref_sample_tokens)
            line["cpu_baseline"] = {"value": m["rate_1core"], "unit": "tokens/s", "cores": 1, "kind": "reference",
                                    "sample": _sample_text(cfg, args.ref_sample_tokens, m)}
        except Exception as e:  # the checker is optional on the bench line
            line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if args.profile_json and rank == 0:
        pathlib.Path(args.profile_json).write_text(json.dumps({"profile": prof, "line": line}, indent=1))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
