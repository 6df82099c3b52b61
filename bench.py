"""bench.py — MemFine chunked MoE layer, forward + backward tokens/s on B200.

Contract (driver): ``python bench.py --gpus N --steps K --warmup W`` (torchrun for N > 1,
one rank per GPU, EP = N) prints ONE JSON line on rank 0.

Workload (BASELINE.json configs[1], the config its metric is quoted on): the Mixtral-8x7B-
style layer — 8 experts, top-2, h = 4096, SwiGLU FFN 14336, 16K tokens per GPU, bf16
storage / fp32 accumulation — with Zipf(1.2)-skewed synthetic routing (random popularity
placement).  At N GPUs the experts are split EP = N ways and every rank holds its own 16K
tokens (weak scaling).  One step = memfine_route_counts -> memfine_plan (the forward C: device
tuner, paper model, rule EXACT; the backward C: exact backward workspace) -> memfine_moe_fwd ->
memfine_moe_bwd, all inside the timed region.  `--gpus N` outside torchrun re-launches itself
under torch.distributed.run with N ranks.

``--impl reference`` times the CPU oracle (oracle/, fp64, the method's reference
definition) on a bounded sample of the same workload — the reference arm of this tier.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "MoE layer fwd+bwd tokens/s"
# Algorithmic FLOPs per routed copy and kernel class, in units of h*g:
# gate/up runs in the forward and again as the backward recompute (4+4), down 2, dA 2,
# dX 4, dW_down 2, dW_gate||dW_up 4  -> 22 h g per copy.
FLOP_COEF = {"gemm_gateup_swiglu": 8, "gemm_down": 2, "gemm_dact_epilogue": 2, "gemm_dx": 4,
             "gemm_wgrad_down": 2, "gemm_wgrad_gateup": 4}


def paper_context(per_C, peak_gb):
    """The paper's headline numbers with the hardware it states (context, not the target), beside this run's
    analogues: Method 1 = no chunking (C = 1; the expert activations are recomputed in the backward either way),
    Method 2 = fixed c_k = 8, MACT's c_k = 2 (what MACT picked for both of the paper's models, Table 4)."""
    paper = {"activation_reduction_pct": 48.03, "throughput_vs_method1_pct": 4.42,
             "method2_vs_method1_pct": -5.40, "method3_vs_method2_pct_model1": 18.26,
             "setup": "32 GPUs with 64 GB each (model unnamed), two reduced-layer DeepSeek-V3-based models, "
                      "t=1 p=4 e=32, BF16, Megatron-LM (PAPER.md:209, 232, 238)"}
    this = {}
    try:
        ms = {int(c): v["ms_per_step"] for c, v in per_C.items() if "ms_per_step" in v}
        if 1 in ms and 2 in ms:
            this["activation_reduction_pct_c2"] = 100.0 * (1.0 - peak_gb(2) / peak_gb(1))
            this["throughput_c2_vs_c1_pct"] = 100.0 * (ms[1] / ms[2] - 1.0)
        if 1 in ms and 8 in ms:
            this["activation_reduction_pct_c8"] = 100.0 * (1.0 - peak_gb(8) / peak_gb(1))
            this["throughput_c8_vs_c1_pct"] = 100.0 * (ms[1] / ms[8] - 1.0)
        if 2 in ms and 8 in ms:
            this["throughput_c2_vs_c8_pct"] = 100.0 * (ms[8] / ms[2] - 1.0)
    except Exception as ex:  # noqa: BLE001
        this = {"error": f"{type(ex).__name__}: {ex}"[:200]}
    return {"paper": paper, "this_run": this}


def load_traffic():
    """DRAM bytes per launch per kernel class from the committed ncu capture (tools/ncu_traffic.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_traffic.json")))
    if not files:
        return None, None
    return json.load(open(files[-1])), os.path.relpath(files[-1], ROOT)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
                pw.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "power_w_median": statistics.median(pw) if pw else None, "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # the communicators' init lines (nranks) on stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v: float, world: int) -> float:
    if world == 1:
        return v
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def device_weights(experts, h, g, dev):
    """Seeded per-global-expert weights generated on the device (same recipe as synth)."""
    out = []
    for e in experts:
        gen = torch.Generator(device=dev).manual_seed(7000 + int(e))
        wg = (torch.randn(g, h, generator=gen, device=dev) / math.sqrt(h)).to(torch.bfloat16)
        wu = (torch.randn(g, h, generator=gen, device=dev) / math.sqrt(h)).to(torch.bfloat16)
        wd = (torch.randn(h, g, generator=gen, device=dev) / math.sqrt(g)).to(torch.bfloat16)
        out.append((wg, wu, wd))
    return tuple(torch.stack([o[i] for o in out]).contiguous() for i in range(3))


def step_roofline(counts_h, h, g, k, T, El, C, ms, peaks, nvlink_gbs=900.0):
    """The north star's roofline of a whole step, from the all-gathered counts
    [EP][nsub][E]: per rank r, F_r = 22 h g s''_r FLOPs (fwd 6 + recompute 4 + bwd 12), P_r = 10 (k+1) h T
    bytes of permute traffic (bf16), N_r = 10 h max(off-rank copies sent, received) bytes over NVLink;
    t_roof = max_r max(F_r / tensor peak, P_r / HBM, N_r / NVLink).  t_roof4 adds the chunked method's
    own HBM term W_r = C (8/3)|W_r| + (4C - 2)|W_r| (weights re-read per chunk, fp32 dW written once
    and read-modify-written per later chunk; |W_r| = the rank's bf16 expert weights)."""
    ch = counts_h.to(torch.int64)
    EP = ch.shape[0]
    per_dst = ch.sum(dim=1)                            # [src][E]
    own = [int(per_dst[r, r * El:(r + 1) * El].sum()) for r in range(EP)]
    sent = [int(per_dst[r].sum()) - own[r] for r in range(EP)]
    recv = [int(per_dst[:, r * El:(r + 1) * El].sum()) - own[r] for r in range(EP)]
    s_dd = [int(per_dst[:, r * El:(r + 1) * El].sum()) for r in range(EP)]
    W_r = 3 * El * h * g * 2
    terms = []
    for r in range(EP):
        F = 22.0 * h * g * s_dd[r]
        P = 10.0 * (k + 1) * h * T
        N = 10.0 * h * max(sent[r], recv[r])
        Wb = C * (8.0 / 3.0) * W_r + (4 * C - 2) * W_r
        terms.append((F / (peaks["bf16_tflops_sustained"] * 1e12), P / (peaks["hbm_gbs"] * 1e9),
                      N / (nvlink_gbs * 1e9), (P + Wb) / (peaks["hbm_gbs"] * 1e9)))
    t_roof = max(max(t[0], t[1], t[2]) for t in terms)
    t_roof4 = max(max(t[0], t[3], t[2]) for t in terms)
    # the same terms with the tensor-bound and HBM-bound work NOT overlapped (what a step that runs
    # its dW read-modify-writes and weight re-reads between the GEMMs can reach at best)
    t_serial = max(t[0] + t[3] + t[2] for t in terms)
    hot = max(range(EP), key=lambda r: max(terms[r][:3]))
    return {"t_roof_ms": t_roof * 1e3, "t_roof4_ms": t_roof4 * 1e3, "frac": t_roof / (ms / 1e3),
            "frac4": t_roof4 / (ms / 1e3), "t_serial_ms": t_serial * 1e3, "frac_serial": t_serial / (ms / 1e3),
            "hot_rank": hot,
            "bound": ["tensor", "hbm", "nvlink"][max(range(3), key=lambda i: terms[hot][i])],
            "terms_ms_hot_rank": {"gemm_flops": terms[hot][0] * 1e3, "permute_bytes": terms[hot][1] * 1e3,
                                  "a2a_bytes": terms[hot][2] * 1e3, "permute_plus_weights": terms[hot][3] * 1e3},
            "peaks": {"tensor_tflops": peaks["bf16_tflops_sustained"], "hbm_gbs": peaks["hbm_gbs"],
                      "nvlink_gbs": nvlink_gbs}}


def per_c_roofline(counts_h, h, g, k, T, El, C, ms, peaks):
    """The per-C entry's roofline: t_roof4 (tensor and the chunked method's HBM bytes overlapped, the
    lower bound) and t_serial (not overlapped), both from step_roofline."""
    r = step_roofline(counts_h, h, g, k, T, El, C, ms, peaks)
    return {"t_roof4_ms": r["t_roof4_ms"], "frac4": r["frac4"], "t_serial_ms": r["t_serial_ms"],
            "frac_serial": r["frac_serial"], "hbm_ms_hot_rank": r["terms_ms_hot_rank"]["permute_plus_weights"]}


# ------------------------------------------------------------------------------------ oracle legs
def oracle_sample_time(cfg, ntok: int, rank: int = 0):
    """Oracle (fp64, unchunked Eq. 4 + Eq. 5) fwd + bwd on ntok tokens of the workload; seconds."""
    import oracle
    oracle.build()
    x = synth.make_x(ntok, cfg.h, rank=rank)
    dy = synth.make_dy(ntok, cfg.h, rank=rank)
    ids, w = synth.make_routing(ntok, cfg.E, cfg.k, rank=rank, zipf_s=cfg.zipf_s, placement=cfg.placement)
    wg, wu, wd = synth.make_experts(range(cfg.E), cfg.h, cfg.g)
    b = lambda a: a.contiguous().view(torch.int16).numpy().view(np.uint16)
    d = oracle.Dims(T=ntok, h=cfg.h, g=cfg.g, E=cfg.E, k=cfg.k, in_dtype="bf16")
    args = (b(x), ids, w.astype(np.float64), b(wg), b(wu), b(wd))
    t0 = time.perf_counter()
    oracle.moe_forward(d, *args)
    oracle.moe_backward(d, b(dy), *args)
    return time.perf_counter() - t0, int(oracle.lib().oracle_num_threads())


def cpu_baseline(cfg, ntok: int):
    dt, cores = oracle_sample_time(cfg, ntok)
    return {"value": ntok / dt, "unit": "tokens/s", "cores": cores, "kind": "oracle",
            "sample": f"{ntok} tokens of the {cfg.name} layer (all {cfg.E} experts, full h={cfg.h}, g={cfg.g}), "
                      f"oracle fwd (Eq. 4) + bwd (Eq. 5) incl. dW, fp64, {dt:.1f} s; cost linear in tokens "
                      f"plus a fixed dW zeroing term"}


def emulated_config(args):
    """The config, or with --ep-emulate R one rank's expert load at EP=R: the same T tokens x top-k
    copies routed over E/R experts (the GEMM shapes of a uniform EP=R share; the skew differs)."""
    cfg = synth.CONFIGS[args.config]
    if args.ep_emulate > 1:
        import dataclasses
        assert cfg.E % args.ep_emulate == 0
        El = cfg.E // args.ep_emulate
        if cfg.k <= El:
            cfg = dataclasses.replace(cfg, E=El)
        else:
            # fewer local experts than top-k (Mixtral at EP = 8: one expert per rank): the same T k copies as
            # T k / k' tokens with top-k' = E_l distinct local experts - identical expert GEMM and weight-gradient
            # shapes; the permute moves the same copies from k/k' times as many token rows
            assert (cfg.T * cfg.k) % El == 0
            cfg = dataclasses.replace(cfg, E=El, k=El, T=cfg.T * cfg.k // El)
    return cfg


def workload_config(cfg, args, world: int) -> dict:
    """The workload both arms are measured on (config.workload of the JSON line)."""
    T = args.tokens or cfg.T
    placement = args.placement or cfg.placement
    k0 = synth.CONFIGS[args.config].k
    emu = (f" [one rank's load at EP={args.ep_emulate}: {T}x{cfg.k} copies over E/{args.ep_emulate}="
           f"{cfg.E} local experts, run at EP=1"
           + (f"; top-{k0} routing over {cfg.E} local expert(s) emulated as {T} tokens top-{cfg.k}" if cfg.k != k0
              else "") + "]") if args.ep_emulate > 1 else ""
    T_tok = T * cfg.k // k0
    return {"workload": f"{cfg.name}-style MoE layer: E={cfg.E * args.ep_emulate} top-{k0} h={cfg.h} SwiGLU "
                        f"ffn={cfg.g}, {T_tok} tokens/GPU, Zipf({cfg.zipf_s}) routing ({placement} placement), "
                        f"EP={world}{emu}",
            "tokens_per_gpu": T_tok, "ep": world}


def run_reference(args):
    """The reference arm: the CPU oracle on rank 0 (the other ranks contribute no work); under torchrun
    the ranks meet in a gloo group (CPU) for the barrier and the max over ranks of the timed region."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    cfg = emulated_config(args)
    ntok = args.ref_tokens
    times = []
    cores = None
    if rank == 0:
        for i in range(args.warmup + args.steps):
            dt, cores = oracle_sample_time(cfg, ntok, rank=i % 8)
            if i >= args.warmup:
                times.append(dt)
    ms = 1000.0 * statistics.mean(times) if times else 0.0
    if dist is not None:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.destroy_process_group()
    if rank != 0:
        return
    value = ntok / (ms / 1000.0)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": max(world, args.gpus),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args, max(world, args.gpus)),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": f"{ntok} tokens of the workload per step (all {cfg.E} experts, full "
                                       f"h={cfg.h}, g={cfg.g}), oracle fwd (Eq. 4) + bwd (Eq. 5) incl. dW, fp64; "
                                       f"cost linear in tokens"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(argv, n: int) -> int:
    """`python bench.py --gpus N` outside torchrun: re-run this script under torch.distributed.run with N
    ranks on this node (rendezvous on 127.0.0.1, a free port); the ranks' output passes through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")        # keep NCCL's communicator init lines (nranks) in the log
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="memfine", choices=["memfine", "reference"])
    ap.add_argument("--config", default="mixtral", choices=sorted(synth.CONFIGS))
    ap.add_argument("--tokens", type=int, default=0, help="tokens per GPU (default: the config's)")
    ap.add_argument("--budget-gb", type=float, default=0.0, help="M^GPU for MACT (default: this GPU's HBM)")
    ap.add_argument("--alpha", type=float, default=0.9)
    ap.add_argument("--chunks", type=int, default=0, help="override the tuner's C")
    ap.add_argument("--sweep", type=int, default=1, help="also time every bin C (N=1 only)")
    ap.add_argument("--cpu-tokens", type=int, default=96, help="cpu_baseline sample (~15 s of oracle work on 16 cores)")
    ap.add_argument("--ref-tokens", type=int, default=16,
                    help="reference arm: tokens per step (the oracle's fixed dW work is ~3 s; 16 tokens ~4 s more)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--placement", default=None)
    ap.add_argument("--ep-emulate", type=int, default=1,
                    help="N=1 only: one rank's expert load at EP=R (T*k copies over E/R local experts); "
                         "labelled in config.workload, never the headline")
    ap.add_argument("--mx", type=int, default=1, help="also time the MXFP8 variant (SURVEY N4; N=1 only)")
    ap.add_argument("--overlap", type=int, default=1,
                    help="N>1, C>1: MEMFINE_FLAG_OVERLAP (chunk j+-1's exchange on a comm stream under chunk j's GEMMs)")
    ap.add_argument("--comm-sms", type=int, default=0, help="with --overlap: SMs the GEMMs leave to the comm stream")
    ap.add_argument("--ep-transport", default="copy", choices=["copy", "p2p"],
                    help="N>1: 'copy' = permute into send buffers + NCCL all-to-allv; 'p2p' = dispatch/combine "
                         "fused into the permute kernel and the GEMM epilogues over CUDA-IPC peer memory")
    ap.add_argument("--fixed-c", action="store_true",
                    help="skip the per-step MACT tuner calls (route_counts + plan) inside the timed step")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(sys.argv[1:], args.gpus))
    if args.impl == "reference":
        return run_reference(args)

    from paper_2511_21431_b200 import capi, layer
    world, rank, local = dist_setup()
    assert world == args.gpus or args.gpus == 1 and world == 1, "run N>1 under torchrun"
    dev = torch.device("cuda", local)
    cfg = emulated_config(args)
    placement = args.placement or cfg.placement
    T = args.tokens or cfg.T
    # tokens/s counts the workload's own tokens: an EP emulation that runs T k copies as T k / k' top-k' tokens
    # (fewer local experts than top-k) still processes the copies of T k' / k tokens of the real layer
    T_tok = T * cfg.k // synth.CONFIGS[args.config].k
    EP = world
    assert cfg.E % EP == 0
    El = cfg.E // EP
    h, g, E, k = cfg.h, cfg.g, cfg.E, cfg.k
    pg = None
    if world > 1:
        import torch.distributed as dist
        pg = dist.group.WORLD

    # ---------------------------------------------------------------- inputs (seeded, synthetic)
    x_h = synth.make_x(T, h, rank=rank)
    dy_h = synth.make_dy(T, h, rank=rank)
    ids_np, w_np = synth.make_routing(T, E, k, rank=rank, zipf_s=cfg.zipf_s, placement=placement)
    ids_h = torch.from_numpy(ids_np)
    w_h = torch.from_numpy(w_np)
    x, dy, ids, w = (t.to(dev) for t in (x_h, dy_h, ids_h, w_h))
    wg, wu, wd = device_weights(synth.local_experts(E, EP, rank), h, g, dev)
    f32 = dict(dtype=torch.float32, device=dev)
    dwg, dwu, dwd = torch.empty(wg.shape, **f32), torch.empty(wu.shape, **f32), torch.empty(wd.shape, **f32)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    dscore = torch.empty(w.shape, **f32)

    overlap = bool(args.overlap) and world > 1 and args.ep_transport == "copy"
    mf = layer.MemFine(T, h, g, E, k, ep_size=EP, ep_rank=rank, dtype=torch.bfloat16, process_group=pg,
                       overlap=overlap)
    if overlap and args.comm_sms:
        mf.set_comm_sms(args.comm_sms)
    bins = (1, 2, 4, 8)

    # ---------------------------------------------------------------- MACT: counts -> C (device tuner)
    counts = mf.route_counts(ids, nsub=8)
    torch.cuda.synchronize()
    counts_h = counts.cpu()
    cap = int(args.budget_gb * 1e9) if args.budget_gb else torch.cuda.get_device_properties(dev).total_memory
    static = sum(t.numel() * t.element_size() for t in (wg, wu, wd, dwg, dwu, dwd, x, dy, y, dx, ids, w, dscore))
    # forward C: the paper's model (Eqs. 8-9, beta = D_t (2h + 2g)) with rule EXACT (the library default);
    # backward C: the exact backward workspace (model IMPL, pass BWD), whose live set per row is larger
    budget_f = capi.make_budget(cap, args.alpha, static, 0, bins=bins)
    budget_b = capi.make_budget(cap, args.alpha, static, 0, bins=bins, model=capi.MODEL_IMPL, pass_=capi.BWD)
    plan_f = layer.plan(counts, mf.dims, budget_f)
    plan_b = layer.plan(counts, mf.dims, budget_b)
    assert plan_f["status"] == 0 and plan_b["status"] == 0, (plan_f, plan_b)
    C_f = args.chunks or plan_f["C"]
    C_b = args.chunks or plan_b["C"]
    C = C_b            # the chunked backward is the step's dominant part: reported as config.chunks

    def ws_for(Cc, Cb=None):
        fwd = layer.workspace_bytes(counts_h, mf.dims, Cc, capi.FWD)
        bwd = layer.workspace_bytes(counts_h, mf.dims, Cb or Cc, capi.BWD)
        return fwd, bwd

    def tune_on(idss, stream):
        """A3 inside every step, as a training step runs it: counts (A1 + the A2 all-gather), then the
        device tuner (forward C) and the exact-workspace planner (backward C), in `stream`'s order (only
        that stream is synchronised)."""
        cnt = mf.route_counts(idss, nsub=8, stream=stream)
        cf = args.chunks or layer.plan(cnt, mf.dims, budget_f, stream=stream)["C"]
        cb = args.chunks or layer.plan(cnt, mf.dims, budget_b, stream=stream)["C"]
        return cf, cb

    def tune(idss):
        return tune_on(idss, torch.cuda.current_stream())

    def make_step(Cc, ws, Cb=None, tuned=False):
        def step(xx=x, dyy=dy, idss=ids, ww=w):
            cf, cb = Cc, Cb or Cc
            if tuned:
                cf, cb = tune(idss)
                assert (cf, cb) == (Cc, Cb or Cc)      # fixed inputs: the tuner's choice is fixed too
            mf.moe_fwd(xx, idss, ww, wg, wu, wd, cf, ws, y=y)
            mf.moe_bwd(dyy, xx, idss, ww, wg, wu, wd, cb, ws, dx=dx, dw_gate=dwg, dw_up=dwu, dw_down=dwd,
                       dscore=dscore)
        return step

    def timed(step, K, W, prof=False):
        for _ in range(W):
            step()
        torch.cuda.synchronize()
        st = mf.sync()
        assert st == 0, capi.status_str(st)
        if prof:
            mf.profile_read()
            mf.profile_enable(True)
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            step()
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
        ms = e0.elapsed_time(e1) / K
        profd = None
        if prof:
            profd = mf.profile_read()
            mf.profile_enable(False)
        st = mf.sync()
        assert st == 0, capi.status_str(st)
        return max_over_ranks(ms, world), profd

    fwd_b, bwd_b = ws_for(C_f, C_b)
    ws_bytes = max(fwd_b, bwd_b)
    if world > 1 and args.ep_transport == "p2p":
        # the fused exchange derives every peer's buffer addresses from one workspace size: the largest any
        # rank needs (the counts are all-gathered, so every rank computes the same number)
        for rr in range(world):
            dr = layer.make_dims(T, h, g, E, k, ep_size=EP, ep_rank=rr, dtype=torch.bfloat16)
            ws_bytes = max(ws_bytes, layer.workspace_bytes(counts_h, dr, C_f, capi.FWD),
                           layer.workspace_bytes(counts_h, dr, C_b, capi.BWD))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    if world > 1 and args.ep_transport == "p2p":
        mf.set_ep_transport(capi.EP_P2P)
        mf.register_workspace(ws)
    step = make_step(C_f, ws, C_b, tuned=not args.fixed_c)

    # launches per step (the library's own kernels: the tuner's histogram + plan kernel, fwd, bwd)
    step()
    torch.cuda.synchronize()
    mf.sync()
    launches_fwd_bwd = None
    mf.moe_fwd(x, ids, w, wg, wu, wd, C_f, ws, y=y)
    mf.sync()
    fstats = mf.last_stats()
    lf = fstats["kernel_launches"]
    mf.moe_bwd(dy, x, ids, w, wg, wu, wd, C_b, ws, dx=dx, dw_gate=dwg, dw_up=dwu, dw_down=dwd, dscore=dscore)
    mf.sync()
    bstats = mf.last_stats()
    launches_fwd_bwd = lf + bstats["kernel_launches"] + (0 if args.fixed_c else 2)
    rows_total = sum(bstats["rows"])  # s''_r: copies this rank's experts processed per step
    comm_ops = {"fwd": fstats.get("comm_ops", 0), "bwd": bstats.get("comm_ops", 0),
                "per_chunk_fwd": fstats.get("comm_ops", 0) / C_f, "per_chunk_bwd": bstats.get("comm_ops", 0) / C_b}

    with ClockSampler(local) as clk:
        ms, prof = timed(step, args.steps, args.warmup, prof=True)
        # the same timed region again without event bracketing (the headline number)
        ms_plain, _ = timed(step, args.steps, 1, prof=False)
    ms = ms_plain
    value = EP * T_tok / (ms / 1000.0)

    # ---------------------------------------------------------------- roofline of the dominant kernel
    peaks = load_peaks()
    dom = max(prof, key=lambda s: prof[s]["ms"])
    tot_ms = sum(v["ms"] for v in prof.values())
    roof = None
    if dom in FLOP_COEF and prof[dom]["launches"]:
        flops_step = FLOP_COEF[dom] * h * g * rows_total
        per_launch_flops = flops_step * args.steps / prof[dom]["launches"]
        avg_ms = prof[dom]["ms"] / prof[dom]["launches"]
        achieved = per_launch_flops / (avg_ms / 1000.0) / 1e12
        # the sustained peak for a kernel inside a long step at the power cap; a short step that never reaches
        # the capped clock can run its GEMMs above it - then the burst figure is the ceiling that applies
        burst = achieved > peaks["bf16_tflops_sustained"]
        peak = peaks["bf16_tflops"] if burst else peaks["bf16_tflops_sustained"]
        traffic, tsrc = load_traffic()
        # the committed capture is of the default workload (Mixtral, EP = 1, C = 1); other shapes: null
        same = (args.config == "mixtral" and args.ep_emulate == 1 and not args.tokens and world == 1 and C == 1)
        tb = traffic.get(dom, {}).get("bytes_per_launch") if (traffic and same) else None
        roof = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": tb,
                "traffic_source": f"{tsrc}: ncu --set full dram__bytes_read.sum + dram__bytes_write.sum per launch"
                if tb else None,
                "algorithmic_flops_per_launch": per_launch_flops,
                "peak_source": (f"{peaks['source']} bf16_tflops (burst: the kernel ran above the sustained rate, "
                                "the step did not reach the power-capped clock)") if burst else
                               f"{peaks['source']} bf16_tflops_sustained (kernel timed inside a long step)",
                "share_of_step": prof[dom]["ms"] / tot_ms if tot_ms else None}
    elif dom in ("dispatch_permute", "combine_unpermute") and prof[dom]["launches"]:
        # HBM-bound permute kernels (small layers): algorithmic bytes per step, bf16 rows of h.
        # dispatch: fwd reads T rows of x and writes s'' rows, bwd the same for x and dY;
        # combine: fwd reads s'' rows of o and writes T rows of y, bwd the same for dX.
        eb = 2 * h
        bytes_step = (3 * T + 3 * rows_total) * eb if dom == "dispatch_permute" else (2 * rows_total + 2 * T) * eb
        per_launch = bytes_step * args.steps / prof[dom]["launches"]
        avg_ms = prof[dom]["ms"] / prof[dom]["launches"]
        achieved = per_launch / (avg_ms / 1000.0) / 1e9
        peak = peaks["hbm_gbs"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None,
                "algorithmic_bytes_per_launch": per_launch,
                "peak_source": f"{peaks['source']} hbm_gbs (copy)",
                "share_of_step": prof[dom]["ms"] / tot_ms if tot_ms else None}
    gemm_ms = sum(prof[s]["ms"] for s in FLOP_COEF) / args.steps
    all_gemm_tflops = 22 * h * g * rows_total / (gemm_ms / 1000.0) / 1e12 if gemm_ms else None
    step_tflops = 22 * h * g * rows_total / (ms / 1000.0) / 1e12

    step_roof = step_roofline(counts_h, h, g, k, T, El, C, ms, peaks)

    # ---------------------------------------------------------------- e2e through the public API
    # Every step copies its inputs (x, dY, ids, scores) host->device from pinned memory and reads
    # its results (y, dX) device->host, inside the timed region.  Inputs and results are double-buffered
    # and move on two copy streams (one per direction: the H2D and D2H copy engines run concurrently):
    # step i+2's inputs land and step i's results leave while step i+1 computes.
    pin = lambda t: t.pin_memory()
    xh, dyh, idsh, wh = pin(x_h), pin(dy_h), pin(ids_h), pin(w_h)
    out_h = [(torch.empty(y.shape, dtype=y.dtype).pin_memory(), torch.empty(dx.shape, dtype=dx.dtype).pin_memory())
             for _ in range(2)]
    ins = [tuple(torch.empty_like(t) for t in (x, dy, ids, w)) for _ in range(2)]
    outs = [(y, dx), (torch.empty_like(y), torch.empty_like(dx))]
    cs_in = torch.cuda.Stream()    # H2D
    cs_out = torch.cuda.Stream()   # D2H
    ts = torch.cuda.Stream()
    comp = torch.cuda.current_stream()

    def e2e_run(K):
        in_ready = [torch.cuda.Event() for _ in range(2)]    # buffer b's inputs landed
        done = [torch.cuda.Event() for _ in range(2)]        # the step using buffer b finished
        out_read = [torch.cuda.Event() for _ in range(2)]    # buffer b's results left the device
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        cs_in.wait_stream(comp)
        cs_out.wait_stream(comp)

        def h2d(b, after=None):
            with torch.cuda.stream(cs_in):
                if after is not None:
                    cs_in.wait_event(after)   # the step that read ins[b] before has finished
                for dst, src in zip(ins[b], (xh, dyh, idsh, wh)):
                    dst.copy_(src, non_blocking=True)
                in_ready[b].record(cs_in)

        # EP = 1: step i+1's tuner (route_counts + plan) runs on its own stream as soon as its ids have
        # landed, while step i computes, so the host's wait for C never leaves the GPU idle.  EP > 1: the
        # count all-gather shares the NCCL communicator with the step's exchanges, so it stays in order
        # on the compute stream.
        ahead = world == 1 and not args.fixed_c

        def plan_ahead(b):
            ts.wait_event(in_ready[b])
            with torch.cuda.stream(ts):
                return tune_on(ins[b][2], ts)

        h2d(0)
        if K > 1:
            h2d(1)
        nxt = plan_ahead(0) if ahead else None
        for i in range(K):
            b = i % 2
            comp.wait_event(in_ready[b])
            if i >= 2:
                comp.wait_event(out_read[b])   # step i-2's results have left outs[b]
            xx, dyy, idd, ww = ins[b]
            yy, dxx = outs[b]
            if args.fixed_c:
                cf, cb = C_f, C_b
            elif ahead:
                cf, cb = nxt
                comp.wait_stream(ts)    # (the counts were read on ts)
            else:
                cf, cb = tune(idd)
            mf.moe_fwd(xx, idd, ww, wg, wu, wd, cf, ws, y=yy)
            mf.moe_bwd(dyy, xx, idd, ww, wg, wu, wd, cb, ws, dx=dxx, dw_gate=dwg, dw_up=dwu, dw_down=dwd,
                       dscore=dscore)
            done[b].record(comp)
            with torch.cuda.stream(cs_out):
                cs_out.wait_event(done[b])
                out_h[b][0].copy_(yy, non_blocking=True)
                out_h[b][1].copy_(dxx, non_blocking=True)
                out_read[b].record(cs_out)
            if i + 2 < K:
                h2d(b, after=done[b])
            if ahead and i + 1 < K:
                nxt = plan_ahead((i + 1) % 2)
        comp.wait_stream(cs_out)
        comp.wait_stream(cs_in)
        e1.record(comp)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    e2e_run(2)
    mf.sync()
    barrier(world)
    ms_e2e = max_over_ranks(e2e_run(args.steps), world)
    assert mf.sync() == 0
    h2d = sum(t.numel() * t.element_size() for t in (xh, dyh, idsh, wh))
    d2h = sum(t.numel() * t.element_size() for t in out_h[0])

    # ---------------------------------------------------------------- memory: peak activation vs unchunked
    def peak_gb(Cc):
        f, b = ws_for(Cc)
        return max(f, b) / 1e9

    per_C = {}
    if args.sweep and world == 1:
        for Cc in bins:
            if Cc == C_f == C_b:
                per_C[Cc] = {"ms_per_step": ms, "tokens_per_s": value, "peak_act_gb": peak_gb(Cc),
                             "roofline": per_c_roofline(counts_h, h, g, k, T, El, Cc, ms, peaks)}
                continue
            try:   # a side measurement: a failure here must not cost the headline line
                wsc = torch.empty(int(peak_gb(Cc) * 1e9) + 1, dtype=torch.uint8, device=dev)
                msc, _ = timed(make_step(Cc, wsc), max(3, args.steps // 2), 1)
                per_C[Cc] = {"ms_per_step": msc, "tokens_per_s": EP * T_tok / (msc / 1000.0), "peak_act_gb": peak_gb(Cc),
                             "roofline": per_c_roofline(counts_h, h, g, k, T, El, Cc, msc, peaks)}
                del wsc
            except Exception as ex:  # noqa: BLE001
                per_C[Cc] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
                torch.cuda.synchronize()
    peak_c = max(fwd_b, bwd_b) / 1e9
    peak_1 = peak_gb(1)
    beta = 2 * (2 * h + 2 * g)
    paper_model = {Cc: beta * max(int(counts_h[:, j * (8 // Cc):(j + 1) * (8 // Cc), rank * El:(rank + 1) * El].sum())
                                  for j in range(Cc)) / 1e9 for Cc in bins}

    # ---------------------------------------------------------------- MXFP8 variant (N4, reading R28)
    # Same workload and C; the weights are re-quantised inside every timed step (they change
    # every training step).  Reported beside the BF16 headline, never as it.
    variants = {}
    if args.mx and world == 1 and h % 128 == 0 and g % 128 == 0:
        y_bf16 = y.float().clone()
        for vname, mxw in (("mxfp8", False), ("mxfp8_wgrad", True)):
            try:   # side measurements: a failure here must not cost the headline line
                mfx = layer.MemFine(T, h, g, E, k, mx=True, mx_wgrad=mxw)
                wq = torch.empty(layer.mx_weights_bytes(mfx.dims), dtype=torch.uint8, device=dev)
                fb = layer.workspace_bytes(counts_h, mfx.dims, C, capi.FWD)
                bb = layer.workspace_bytes(counts_h, mfx.dims, C, capi.BWD)
                wsx = torch.empty(max(fb, bb), dtype=torch.uint8, device=dev)

                def step_mx():
                    mfx.mx_quantize_weights(wg, wu, wd, wq=wq)
                    mfx.moe_fwd(x, ids, w, wg, wu, wd, C, wsx, y=y)
                    mfx.moe_bwd(dy, x, ids, w, wg, wu, wd, C, wsx, dx=dx, dw_gate=dwg, dw_up=dwu, dw_down=dwd,
                                dscore=dscore)

                for _ in range(args.warmup):
                    step_mx()
                torch.cuda.synchronize()
                assert mfx.sync() == 0
                mfx.profile_read()
                mfx.profile_enable(True)
                for _ in range(2):
                    step_mx()
                torch.cuda.synchronize()
                profx = mfx.profile_read()
                mfx.profile_enable(False)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(args.steps):
                    step_mx()
                e1.record()
                torch.cuda.synchronize()
                assert mfx.sync() == 0
                msx = e0.elapsed_time(e1) / args.steps
                mfx.moe_fwd(x, ids, w, wg, wu, wd, C, wsx, y=y)
                torch.cuda.synchronize()
                dev_y = float((y.float() - y_bf16).abs().max() / y_bf16.abs().max())
                variants[vname] = {
                    "ms_per_step": msx, "tokens_per_s": EP * T_tok / (msx / 1000.0),
                    "speedup_vs_bf16": ms / msx,
                    "operands": "E4M3 + E8M0 scale per 32 along K (tcgen05 kind::mxf8f6f4.block_scale) for gate/up, "
                                "down and dX" + (" and the weight gradients (columnwise along the copies, reading R28c)"
                                                 if mxw else "; weight gradients bf16") +
                                "; dA bf16; weights re-quantised every step",
                    "y_max_rel_dev_vs_bf16_path": dev_y,
                    "peak_act_gb": max(fb, bb) / 1e9,
                    "kernel_ms_per_step": {s_: v["ms"] / 2 for s_, v in profx.items() if v["launches"]},
                }
                mfx.close()
                del wsx, wq
            except Exception as ex:  # noqa: BLE001
                variants[vname] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
                torch.cuda.synchronize()

    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {**workload_config(cfg, args, world), "chunks": C,
                   "tuner": {"in_timed_step": not args.fixed_c, "rule": "EXACT (library default)",
                             "fwd": {"C": C_f, "model": "paper (Eqs. 8-9, beta = D_t (2h + 2g))", **plan_f},
                             "bwd": {"C": C_b, "model": "IMPL (exact backward workspace)", **plan_b}},
                   "comm_ops": comm_ops,
                   "ep_transport": args.ep_transport if world > 1 else None,
                   "overlap": overlap and C > 1,
                   "pdl": os.environ.get("MEMFINE_PDL", "1") != "0",   # programmatic dependent launch
                   "budget": {"gpu_capacity_bytes": cap, "alpha": args.alpha, "static_bytes": static},
                   "l2": "no flush: every step streams > 126 MB (weights 2.8 GB at EP=1, activations GBs)"},
        "peak_act_gb": peak_c, "peak_act_gb_unchunked": peak_1,
        "peak_act_paper_model_gb": paper_model,
        "per_C": per_C,
        "roofline": roof,
        "step_roofline": step_roof,
        "gemm_tflops_all_kernels": all_gemm_tflops, "step_tflops": step_tflops,
        "kernel_ms_per_step": {s: v["ms"] / args.steps for s, v in prof.items() if v["launches"]},
        "clocks": clk.summary(),
        "e2e": {"value": EP * T_tok / (ms_e2e / 1000.0), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e},
        "gpu_launches": launches_fwd_bwd * args.steps,
        "variants": variants,
        "paper_context": paper_context(per_C, peak_gb),
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_tokens)
        except Exception as ex:  # noqa: BLE001
            line["cpu_baseline"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
