"""MoE-layer tokens/sec of the speculative-token-shuffling layer on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl smoe|reference]
                    [--config mixtral] [--tokens 16384] [--eps 0.2]

A step is one MoE-layer forward (Algorithm 2: lookup/plan -> SRS -> gate ->
A2A dispatch -> SwiGLU grouped GEMM -> down GEMM + A2A combine -> combine +
SAG) over one batch of synthetic tokens.  The workload is BASELINE.json
configs[1] (Mixtral-8x7B layer, 8 experts, top-2, hidden 4096, EP=8): the 8
EP shards are spread over the N GPUs (all 8 on one GPU at N=1, peer buffers
over CUDA IPC / NVLink at N>1), tokens_per_gpu fixed -> weak scaling.

value   = tokens processed by all GPUs / device time (inputs resident in HBM)
e2e     = same metric through SpecMoELayer.forward() with pinned HOST inputs:
          H2D of the partials + ids every step, D2H of the layer output
roofline: the SwiGLU expert GEMM (dominant kernel), CUDA-event timed in the
          timed region, vs the measured bf16 peak in MEASURED_PEAKS.json
cpu_baseline: the CPU oracle port (oracle/layer_ref) on a bounded sample of the
          same workload, on this host's cores
`--impl reference` times that CPU path alone (the reference is pure Python and
ships no layer; its arithmetic is restated in oracle/).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="smoe", choices=["smoe", "reference"])
    p.add_argument("--config", default="mixtral")
    p.add_argument("--tokens", type=int, default=16384, help="tokens per GPU per step")
    p.add_argument("--eps", type=float, default=0.2, help="planted routing noise")
    p.add_argument("--ep", type=int, default=0, help="EP shards (default: config's 8)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU baseline work")
    p.add_argument("--ref-budget", type=float, default=300.0,
                   help="--impl reference: max seconds for the K timed steps")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-dsmoe", action="store_true", help="skip the DS-MoE baseline timing")
    p.add_argument("--no-decode", action="store_true", help="skip the 64-token decode timing")
    p.add_argument("--tune", action="store_true",
                   help="run the init-time up-GEMM schedule choice (SpecMoELayer.tune_gemm_order) "
                        "before the timed region (off by default: its ~25 extra forwards heat "
                        "the GPU and the power cap then lowers the timed region's clock more "
                        "than the schedule gains, profiles/r2/gemm_cg_up/tune_ab.txt)")
    return p.parse_args()


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return {"hbm": d.get("hbm_gbs", 6650.0), "bf16": d.get("bf16_tflops", 1590.0),
                "bf16_sustained": d.get("bf16_tflops_sustained", 1400.0), "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "src": "fallback"}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "25"], stdout=self.fh,
                stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=5)
            self.fh.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        load = [r for r in rows if r[2] > 250.0] or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[3]) if v == "Active"})
        return {"sm_mhz": float(np.median([r[0] for r in load])), "sm_max_mhz": rows[0][1],
                "reasons": reasons, "samples": len(load)}


def cpu_threads() -> int:
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(n)) if n else (os.cpu_count() or 1)
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(bundle, partials, tokens, hist, gate_w, w1, w3, w2, k, budget, n_max,
                  fixed: int | None = None):
    """Time the CPU oracle (oracle/layer_ref) on the first n_s tokens: n_s =
    `fixed` when given, else calibrated so one call costs about `budget`
    seconds (capped at n_max)."""
    from oracle import layer_ref
    tab = bundle

    def run(ns):
        t0 = time.perf_counter()
        layer_ref.layer_forward(partials=partials[:, :ns], tokens=tokens[:ns], hist=hist[:ns],
                                t_labels=tab.token_table.labels,
                                t_conf=tab.token_table.confidence, a_best=tab.ngram_table.best,
                                a_conf=tab.ngram_table.confidence,
                                n_clusters=tab.token_table.n_clusters,
                                expert_labels=np.asarray(tab.expert_labels), gate_w=gate_w,
                                w1=w1, w3=w3, w2=w2, k=k)
        return time.perf_counter() - t0

    if fixed is not None:
        return fixed, run(fixed)
    ns = min(64, n_max)
    t = run(ns)
    ns2 = int(min(n_max, max(ns, ns * budget / max(t, 1e-3))))
    if ns2 > ns:
        t = run(ns2)
        ns = ns2
    return ns, t


def host_copy_weights(w):
    import torch
    f = lambda x: x.float().cpu().numpy() if isinstance(x, torch.Tensor) else x  # noqa: E731
    return f(w.gate_w), f(w.w1), f(w.w3), f(w.w2)


def emit(line: dict):
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- reference arm
def host_workload(args, cfg, n):
    """The bench workload (same generator semantics as synth.make_workload:
    planted routing, orthonormal gate, 1/sqrt(d)-scaled SwiGLU weights) built
    on the HOST for the CPU arms; big tensors from torch's CPU RNG, rounded
    to bf16 values, as float32 numpy arrays."""
    import torch
    from paper_2503_04398_b200 import synth
    G, N, k, d, f, vocab = cfg["G"], cfg["N"], cfg["k"], cfg["d"], cfg["f"], cfg["vocab"]
    rng = np.random.default_rng(args.seed)
    bundle = synth.make_bundle(G, N, vocab, rng)
    tokens = rng.integers(0, vocab, size=n).astype(np.int64)
    cl = np.asarray(bundle.token_table.labels, dtype=np.int64)[tokens]
    hist = rng.integers(0, G, size=(n, 2)).astype(np.int64)
    keep = rng.random(n) < 0.9
    hist[keep] = cl[keep, None]
    chosen = synth.routing_choices(bundle, tokens, k, args.eps, rng)
    gate = synth.planted_gate(N, d, rng)
    g = torch.Generator().manual_seed(args.seed)
    bf = lambda x: x.to(torch.bfloat16).float().numpy()  # noqa: E731
    coef = torch.tensor(1.0 - 0.5 * np.arange(k) / k, dtype=torch.float32)
    gt = torch.from_numpy(gate)
    h = 8.0 * (coef[None, :, None] * gt[torch.from_numpy(chosen)]).sum(1)
    h += 0.05 * torch.randn((n, d), generator=g)
    z = torch.randn((G, n, d), generator=g)
    z -= z.mean(0, keepdim=True)
    partials = bf(h[None] / G + 0.5 * z)
    del h, z
    w1 = bf(torch.randn((N, f, d), generator=g) / d ** 0.5)
    w3 = bf(torch.randn((N, f, d), generator=g) / d ** 0.5)
    w2 = bf(torch.randn((N, d, f), generator=g) / f ** 0.5)
    return bundle, tokens, hist, gate, w1, w3, w2, partials


def run_reference(args, world, rank):
    """The reference's CPU path on the host cores (the reference is pure
    Python and ships no layer: its index half and the fp32 layer are restated
    in oracle/), on the SAME workload as the GPU arm: every
    timed step is the whole batch (tokens_per_gpu x N tokens) unless K steps
    of it would exceed --ref-budget seconds, in which case each step is the
    largest leading sample that fits (config.same_config says which)."""
    if rank != 0:
        return
    import torch
    from paper_2503_04398_b200 import synth
    torch.set_num_threads(os.cpu_count() or 1)
    cfg = dict(synth.CONFIGS[args.config])
    if args.ep:
        cfg["G"] = args.ep
    n_full = args.tokens * max(world, args.gpus)
    bundle, tokens, hist, gate, w1, w3, w2, parts = host_workload(args, cfg, n_full)
    # warm-up + calibration on a small leading sample (untimed)
    n_cal = min(512, n_full)
    t_cal = min(oracle_sample(bundle, parts, tokens, hist, gate, w1, w3, w2, cfg["k"], 0.0,
                              n_cal, fixed=n_cal)[1] for _ in range(max(1, args.warmup)))
    per_tok = t_cal / n_cal
    ns = n_full
    if args.steps * per_tok * n_full > args.ref_budget:
        ns = int(max(n_cal, min(n_full, args.ref_budget / args.steps / per_tok)))
    times = []
    for _ in range(args.steps):
        times.append(oracle_sample(bundle, parts, tokens, hist, gate, w1, w3, w2, cfg["k"], 0.0,
                                   ns, fixed=ns)[1])
    total = sum(times)
    value = ns * len(times) / total
    cores = cpu_threads()
    same = ns == n_full
    emit({"impl": "reference", "metric": "MoE-layer tokens/sec", "value": value,
          "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
          "ms_per_step": 1e3 * total / len(times), "higher_is_better": True, "scaling": "weak",
          "vs_baseline": None, "dtype": "f32", "data": "synthetic (planted skew, host RNG)",
          "config": {"workload": f"{args.config} MoE layer (N={cfg['N']} experts, top-{cfg['k']}, "
                                 f"hidden {cfg['d']}, ffn {cfg['f']}), EP={cfg['G']} shards",
                     "tokens_per_gpu": args.tokens, "global_tokens": n_full,
                     "tokens_per_step": ns, "same_config": same, "eps": args.eps},
          "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "port",
                           "sample": (f"the whole {n_full}-token batch per step" if same else
                                      f"first {ns} of the {n_full}-token batch per step "
                                      f"(--ref-budget {args.ref_budget:.0f} s)") +
                                     f" through oracle/layer_ref (lookup, plan, SRS over "
                                     f"{cfg['G']} partials, fp32 gate, SwiGLU experts, combine)"},
          "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": 0}})


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def ensure_world(args) -> None:
    """`--gpus N` means N ranks, one per GPU.  Launched without torchrun
    (no WORLD_SIZE) and N > 1, re-exec under torch.distributed.run with N
    processes; launched by torchrun with a different world size, fail.  A
    plain `python bench.py --gpus 8` can therefore never silently time N = 1."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None:
        if args.gpus <= 1:
            return
        if args.impl == "smoe" and os.environ.get("SMOE_BENCH_SAME_GPU") != "1":
            import torch
            have = torch.cuda.device_count()
            if have < args.gpus:
                sys.exit(f"bench.py: --gpus {args.gpus} but this box has {have} CUDA device(s)")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(_free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if int(env_world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world}: refusing to time "
                 "a different GPU count than requested")


# --------------------------------------------------------------------------- smoe arm
def main():
    args = parse()
    ensure_world(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    # SMOE_BENCH_SAME_GPU=1 (tests only): every rank on cuda:0 with gloo for the
    # host plumbing, so the multi-process path can be exercised on one GPU.
    same_gpu = os.environ.get("SMOE_BENCH_SAME_GPU") == "1"
    if same_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    from paper_2503_04398_b200 import SpecMoELayer, synth
    from paper_2503_04398_b200 import _native as N

    group = None
    if world > 1:
        import torch.distributed as dist
        if same_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        from paper_2503_04398_b200.dist import ShardGroup
        group = ShardGroup.from_torch_distributed()

    cfg = dict(synth.CONFIGS[args.config])
    if args.ep:
        cfg["G"] = args.ep
    G, k, d, f = cfg["G"], cfg["k"], cfg["d"], cfg["f"]
    n = args.tokens * world                      # weak scaling: tokens per GPU fixed
    w = synth.make_workload(args.config, n=n, eps=args.eps, seed=args.seed, device=True,
                            cfg_override=cfg)
    layer = SpecMoELayer(w.bundle, w.gate_w, w.w1, w.w3, w.w2, top_k=k, max_tokens=n,
                         group=group)
    L = layer.shard_count
    layer.partial_views(n).copy_(w.partials[layer.shard_begin:layer.shard_begin + L])
    tok = torch.as_tensor(w.tokens, device="cuda")
    hist = torch.as_tensor(w.hist, device="cuda")
    stream = torch.cuda.current_stream()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cpu" if same_gpu else "cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---------------- device-resident timed region (value + roofline)
    for _ in range(args.warmup):
        layer.run_device(tok, hist)
    torch.cuda.synchronize()
    layer.check_errors()
    # the library's init-time schedule choice for the up GEMM on this GPU
    # (bit-identical outputs either way; untimed, before the timed region)
    up_schedule = layer.tune_gemm_order(tok, hist) if args.tune else {"tuned": False}
    for _ in range(2):
        layer.run_device(tok, hist)
    torch.cuda.synchronize()
    NS = len(N.STAGE_NAMES)
    # the headline: K whole forwards back to back (the stages chained by
    # programmatic dependent launch, nothing recorded between them)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    torch.cuda.synchronize()
    with Clocks(local_rank) as clk:
        start.record(stream)
        for s in range(args.steps):
            layer.run_device(tok, hist)
        end.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = start.elapsed_time(end)
    # the per-stage breakdown (and the roofline's kernel times): a second pass
    # of K forwards with an event after every stage, captured as ONE CUDA
    # graph (external event nodes) and replayed, so the host's per-stage
    # launch path adds no gaps; events between stages still stop the next
    # stage from launching early, so the stages sum to a little more than the
    # step.  Eager fallback if the capture fails.
    def staged_pass(steps):
        evs = [[torch.cuda.Event(enable_timing=True, external=True) for _ in range(NS + 1)]
               for _ in range(steps)]
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                cs = torch.cuda.current_stream()
                for s_ in range(steps):
                    evs[s_][0].record(cs)
                    for j in range(NS):
                        layer.run_device(tok, hist, stages=[j])
                        evs[s_][j + 1].record(cs)
            barrier()
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            barrier()
            del g
            return evs, "cuda-graph replay, external event nodes between stages"
        except Exception:                   # eager: the same pass from the host
            evs = [[torch.cuda.Event(enable_timing=True) for _ in range(NS + 1)]
                   for _ in range(steps)]
            barrier()
            torch.cuda.synchronize()
            for s_ in range(steps):
                evs[s_][0].record(stream)
                for j in range(NS):
                    layer.run_device(tok, hist, stages=[j])
                    evs[s_][j + 1].record(stream)
            torch.cuda.synchronize()
            barrier()
            return evs, "eager, events between stages"

    ev, stage_timing = staged_pass(args.steps)
    stage_ms = {nm: float(np.mean([ev[s][j].elapsed_time(ev[s][j + 1]) for s in range(args.steps)]))
                for j, nm in enumerate(N.STAGE_NAMES)}
    up_ms, down_ms = stage_ms["expert_up"], stage_ms["expert_down"]
    ms_total = max_over_ranks(ms_total)
    layer.check_errors()
    st = layer.stats(n)
    if world > 1:                        # pair counts of this process's shards -> whole job
        lr = [float(st["local_tokens"]), float(st["remote_tokens"])]
        tot = torch.tensor(lr, device="cpu" if same_gpu else "cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tot)
        st["local_tokens"], st["remote_tokens"] = int(tot[0].item()), int(tot[1].item())
        st["measured_alpha"] = st["local_tokens"] / max(st["local_tokens"] + st["remote_tokens"], 1)
    ms_step = ms_total / args.steps
    value = n * args.steps / (ms_total / 1e3)
    # rows the expert GEMMs of THIS process multiplied = pairs routed to its expert slots
    cm = layer.counts_mat.cpu().numpy()
    e0 = int(layer.slot_first[layer.shard_begin])
    e1 = int(layer.slot_first[layer.shard_begin + layer.shard_count])
    gemm_rows = float(cm[:, e0:e1].sum())
    pk = peaks()
    up_flops = 2.0 * gemm_rows * d * (2 * f)
    down_flops = 2.0 * gemm_rows * f * d
    # per-stage roofline of this process (algorithmic bytes / flops)
    n_loc = float(sum(int(x) for x in layer.plan_counts.cpu().numpy()[
        layer.shard_begin:layer.shard_begin + L]))
    pairs_loc = n_loc * k
    grp = int(layer.group_t.item())
    h = w.hist.shape[1]
    row = 2.0 * d
    stage_bytes = {
        "plan": n * (8 + 8 * h + 12) + 24.0 * n + 8.0 * G * grp,
        "srs": (G + 1) * n_loc * row,
        "gate": n_loc * row + pairs_loc * 8,
        "route": 16.0 * pairs_loc,
        "dispatch": n_loc * row + pairs_loc * (row + 8),
        # one output copy per process (co-resident shards share it)
        "combine_sag": pairs_loc * row + world * n_loc * row + 8 * n_loc,
    }
    stages_rf = []
    for nm in N.STAGE_NAMES:
        t_s = stage_ms[nm] / 1e3
        if nm in ("expert_up", "expert_down"):
            fl = up_flops if nm == "expert_up" else down_flops
            stages_rf.append({"stage": nm, "ms": stage_ms[nm], "bound": "tensor",
                              "algorithmic": fl, "unit": "TFLOP/s",
                              "achieved": fl / t_s / 1e12, "peak": pk["bf16_sustained"],
                              "frac": fl / t_s / 1e12 / pk["bf16_sustained"]})
        else:
            by = stage_bytes[nm]
            stages_rf.append({"stage": nm, "ms": stage_ms[nm],
                              "bound": "latency" if nm in ("plan", "route") else "hbm",
                              "algorithmic": by, "unit": "GB/s", "achieved": by / t_s / 1e9,
                              "peak": pk["hbm"], "frac": by / t_s / 1e9 / pk["hbm"]})
    achieved = up_flops / (up_ms / 1e3) / 1e12
    clocks = clk.summary()

    # ---------------- e2e through the public API with pinned host buffers
    # SpecMoELayer.forward_async: every step H2D-copies its partials / ids /
    # histories from pinned host memory and D2H-copies its output; the copies
    # of neighbouring steps overlap the layer (two steps in flight).
    e2e = None
    if not args.no_e2e:
        host_p = w.partials[layer.shard_begin:layer.shard_begin + L].cpu().pin_memory()
        host_tok = torch.from_numpy(w.tokens).pin_memory()
        host_hist = torch.from_numpy(w.hist).pin_memory()
        outs = [torch.empty((n, d), dtype=torch.bfloat16).pin_memory() for _ in range(2)]

        def run_e2e(steps):
            hs = []
            for i in range(steps):
                if i >= 2:
                    hs[i - 2].result()              # the user consumes step i-2's output
                hs.append(layer.forward_async(host_p, host_tok, host_hist, out=outs[i % 2]))
            for hd in hs[-2:]:
                hd.result()

        run_e2e(3)
        barrier()
        torch.cuda.synchronize()
        ksteps = max(8, args.steps)                # steady state: fill / drain amortised
        # device clock: e0 on an idle GPU before the first H2D is issued, e1
        # after the last D2H has completed (the copy / compute streams all
        # drained by the synchronize), max over ranks
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run_e2e(ksteps)
        torch.cuda.synchronize()
        e1.record(stream)
        e1.synchronize()
        e_ms = max_over_ranks(e0.elapsed_time(e1))
        h2d = host_p.numel() * 2 + host_tok.numel() * 8 + host_hist.numel() * 8
        e2e = {"value": n * ksteps / (e_ms / 1e3), "unit": "tokens/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(n * d * 2),
               "steps": ksteps, "timing": "CUDA events on the device clock, max over ranks",
               "api": "SpecMoELayer.forward_async (pinned host partials/ids/hist in, host "
                      "output out; H2D, layer and D2H of neighbouring steps overlap)"}

    # ---------------- decode-sized batch on the same layer (serving latency)
    # 64 tokens, the whole layer replayed from a CUDA graph (single process);
    # the layer has already run full batches, as a serving loop would have
    decode = None
    if world == 1 and not args.no_decode:
        nd = min(64, n)
        tok_d, hist_d = tok[:nd].clone(), hist[:nd].clone()
        g = layer.capture(tok_d, hist_d)
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 50
        d0.record(stream)
        for _ in range(reps):
            g.replay()
        d1.record(stream)
        torch.cuda.synchronize()
        layer.check_errors()
        us = d0.elapsed_time(d1) / reps * 1e3
        # the experts this batch activates stream their weights once (bf16)
        active = int((np.asarray(layer.stats(nd)["pair_counts"]).sum(0) > 0).sum())
        w_bytes = 2.0 * 3 * active * d * f
        decode = {"tokens": nd, "us_per_step": us, "tokens_per_s": nd / (us / 1e6),
                  "active_experts": active,
                  "weight_stream_roofline_us": w_bytes / (pk["hbm"] * 1e3),
                  "roofline_frac": w_bytes / (pk["hbm"] * 1e3) / us,
                  "mode": "CUDA-graph replay of the whole layer (SpecMoELayer.capture)"}
        del g

    # ---------------- DS-MoE pipeline baseline (AR -> A2A -> A2A -> AG), same kernels
    def timed_stages(lay, run, steps):
        """Whole-step and per-stage device time of `steps` forwards (events
        between stages on the launching stream), max over ranks."""
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(NS + 1)] for _ in range(steps)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for s_ in range(steps):
            evs[s_][0].record(stream)
            for j in range(NS):
                run(stages=[j])
                evs[s_][j + 1].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        per = {nm: max_over_ranks(float(np.mean([evs[s_][j].elapsed_time(evs[s_][j + 1])
                                                 for s_ in range(steps)])))
               for j, nm in enumerate(N.STAGE_NAMES)}
        return max_over_ranks(e0.elapsed_time(e1)), per

    dsm = None
    if not args.no_dsmoe:
        from paper_2503_04398_b200.baseline import DSMoEPipelineLayer
        base = DSMoEPipelineLayer(w.gate_w, w.w1, w.w3, w.w2, n_ranks=G, top_k=k, max_tokens=n,
                                  group=group)
        base.partial_views(n).copy_(w.partials[base.shard_begin:base.shard_begin + L])
        for _ in range(max(2, args.warmup)):
            base.run_device(n=n)
        torch.cuda.synchronize()
        base.check_errors()
        # interleaved rounds (s-MoE, DS-MoE, s-MoE, ...): under the power cap
        # the clock drifts over a run, so timing the two pipelines at
        # different times would compare clocks, not pipelines
        bsteps = max(3, args.steps // 2)
        rounds = 3
        a_ms = b_ms = 0.0
        a_stage = {nm: 0.0 for nm in N.STAGE_NAMES}
        b_stage = {nm: 0.0 for nm in N.STAGE_NAMES}
        for _ in range(rounds):
            t_, per = timed_stages(layer, lambda stages: layer.run_device(tok, hist, stages=stages),
                                   bsteps)
            a_ms += t_
            a_stage = {nm: a_stage[nm] + per[nm] / rounds for nm in N.STAGE_NAMES}
            t_, per = timed_stages(base, lambda stages: base.run_device(n=n, stages=stages),
                                   bsteps)
            b_ms += t_
            b_stage = {nm: b_stage[nm] + per[nm] / rounds for nm in N.STAGE_NAMES}
        base.check_errors()
        layer.check_errors()
        bst = base.stats(n)
        dsm = {"value": n * bsteps * rounds / (b_ms / 1e3), "unit": "tokens/s",
               "ms_per_step": b_ms / (bsteps * rounds),
               "smoe_ms_per_step_interleaved": a_ms / (bsteps * rounds),
               "timing": f"{rounds} interleaved rounds of {bsteps} steps per pipeline",
               "local_activation_rate": bst["measured_alpha"],
               "a2a_bytes_per_step": bst["bytes"]["a2a_dispatch"] + bst["bytes"]["a2a_combine"],
               "stages_ms": b_stage,
               "stage_delta_ms_smoe_minus_dsmoe": {nm: a_stage[nm] - b_stage[nm]
                                                   for nm in N.STAGE_NAMES},
               "impl": "DSMoEPipelineLayer: the s-MoE kernels and runtime with "
                       "SMOE_PIPELINE_DSMOE (two-shot all-reduce + slice instead of SRS, "
                       "combine into all-gather blocks + resume instead of SAG) and "
                       "position-sharding tables (token i -> rank i % G, contiguous experts)",
               "speedup_smoe_over_dsmoe": b_ms / a_ms}
        del base
        torch.cuda.empty_cache()

    # ---------------- CPU baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        gw, w1, w3, w2 = host_copy_weights(w)
        parts = w.partials.float().cpu().numpy()
        ns, t = oracle_sample(w.bundle, parts, w.tokens, w.hist, gw, w1, w3, w2, k,
                              args.cpu_budget, n)
        cpu = {"value": ns / t, "unit": "tokens/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"first {ns} tokens of the step's batch through oracle/layer_ref "
                         f"(lookup, plan, SRS over {G} partials, fp32 gate, SwiGLU, combine)"}

    # plan 2 + srs 1 + gate 1 + route 2 + dispatch 1 + expert GEMMs 2 + combine/SAG 1
    # (+ 5 signal-pad barriers and the deduplicated dispatch's fan-out when
    # shards span processes)
    launches_per_step = 2 + 1 + 1 + 2 + 1 + 2 + 1 + (6 if world > 1 else 0)
    traffic = None
    tf = ROOT / "profiles" / "r2" / "traffic.json"
    if tf.exists():
        t_info = json.loads(tf.read_text())
        c = t_info["config"]
        if (c["workload"], c["tokens_per_gpu"], c["n_gpus"]) == (args.config, args.tokens, world):
            kk = t_info["kernels"]["grouped_gemm_kernel<SwiGLU> (expert up)"]
            traffic = kk["dram_read_bytes"] + kk["dram_write_bytes"]
    if rank == 0:
        emit({"metric": "MoE-layer tokens/sec", "value": value, "unit": "tokens/s",
              "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
              "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
              "vs_baseline": None, "dtype": "bf16", "data": "synthetic (planted skew, seeded)",
              "config": {"workload": f"{args.config} MoE layer (N={cfg['N']} experts, top-{k}, "
                                     f"hidden {d}, ffn {f}), EP={G} shards over {world} GPU(s)",
                         "tokens_per_gpu": args.tokens, "global_tokens": n, "eps": args.eps,
                         "parallelism": f"ep{G}", "l2": "inputs larger than L2 "
                         f"({G * n * d * 2 / 2**20:.0f} MiB partials, "
                         f"{3 * cfg['N'] * d * f * 2 / 2**30:.1f} GiB weights)"},
              "local_activation_rate": st["measured_alpha"],
              "a2a_bytes_per_step": st["bytes"]["a2a_dispatch"] + st["bytes"]["a2a_combine"],
              "stage_bytes": st["bytes"], "group_size": st["group_size"],
              "up_gemm_schedule": up_schedule,
              "stages_ms": stage_ms, "stages_timing": stage_timing,
              "stages_roofline": stages_rf,
              "roofline": {"bound": "tensor", "kernel": "grouped_gemm_kernel<SwiGLU> (expert up)",
                           "achieved": achieved, "peak": pk["bf16_sustained"], "unit": "TFLOP/s",
                           "frac": achieved / pk["bf16_sustained"], "traffic": traffic,
                           "traffic_unit": "bytes per launch (ncu dram read+write)",
                           "algorithmic_bytes": 2 * (gemm_rows * d + 2 * f * d * layer.local_slots
                                                     + gemm_rows * f),
                           "peak_src": pk["src"] + " sustained",
                           "down_gemm_tflops": down_flops / (down_ms / 1e3) / 1e12,
                           "layer_tflops": (up_flops + down_flops) / (ms_step / 1e3) / 1e12},
              "e2e": e2e, "cpu_baseline": cpu, "dsmoe_baseline": dsm, "decode": decode,
              "clocks": clocks,
              "gpu_launches": launches_per_step * args.steps})
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
