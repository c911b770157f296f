#!/usr/bin/env python
"""Benchmark of the FMM evaluation hot path (BASELINE.json metric:
"FMM eval s/step and sustained FP32 TFLOP/s at N particles, 1/2/4/8 B200").

One step = fmm_set_particles (wrap, Morton keys, radix sort, octree) +
fmm_evaluate (P2M, M2M, traversal, M2L, periodic far field, P2P, L2L, L2P,
un-permute): every row of SURVEY 8(a), through the C ABI.

Workload (N = 1): C3 -- Taylor-Green 256^3 = 16.8M particles, periodic
[-pi, pi)^3 with k = 3 image layers, p = 10, theta = 1/2, ncrit = 64 (the
BASELINE config quoted for "full step timing", and the paper's per-GPU size,
P:243/P:284).  Inputs are resident in HBM before the timed region; they are
larger than the 126 MB L2 (470 MB), so no explicit flush is needed.

value = paper-style sustained FP32 TFLOP/s = 174 x (P2P pairs) / step time,
summed over ranks (Table 1 and the flop formula).
e2e   = the same metric with host (pinned) inputs/outputs through the C ABI,
        host<->device copies inside the timed region.

--impl reference times the CPU oracle (test infrastructure) on a bounded
sample of the same workload family.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "FMM eval s/step and sustained FP32 TFLOP/s at N particles, 1/2/4/8 B200"
FLOPS_PER_PAIR = 174          # Table 1: 70 Biot-Savart + 104 stretching
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # 74.4: SMs x FP32 lanes x FMA x max SM clock


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--side", type=int, default=256, help="lattice points per dimension per GPU")
    ap.add_argument("--order", type=int, default=10)
    ap.add_argument("--images", type=int, default=3)
    ap.add_argument("--theta", default="1/2")
    ap.add_argument("--ncrit", type=int, default=64)
    ap.add_argument("--mode", choices=["tiled", "refined", "strong"], default="tiled",
                    help="N > 1: tiled = C5 weak scaling (one 2pi tile of side^3 per GPU, reading Z27); "
                         "refined = the fixed box refined to side*(1..2) per axis; "
                         "strong = C4: one side^3 lattice split over the GPUs by Morton octants")
    ap.add_argument("--partition", choices=["octant", "orb"], default="octant",
                    help="N > 1 with --mode strong: octant = each rank passes its Morton-octant block; orb = "
                         "each rank passes a random 1/N subset and the library redistributes it every step "
                         "(cfg.partition = 1: ORB recursive multisection by a distributed nth-element, NEXT-3)")
    ap.add_argument("--workload", choices=["lattice", "jitter", "advected"], default="lattice",
                    help="N = 1 stress variants of C3 (VERDICT r01): jitter = the lattice jittered by +-h "
                         "(seed 5273); advected = the lattice after one fmm_step (midpoint RK2, dt = 2h, "
                         "max displacement ~2h): leaves gain and lose particles, the tree turns adaptive")
    ap.add_argument("--cpu-fmm-sample", type=int, default=64, help="cpu_baseline: oracle FMM on TG n^3 (C2 = 64)")
    ap.add_argument("--ref-sample", type=int, default=24, help="--impl reference sample: TG n^3 lattice")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def theta_of(s):
    a, b = s.split("/")
    return int(a), int(b)


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi sampled every 200 ms while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "200"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 7:
                self.rows.append(p)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th:
            self.th.join(timeout=5)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------ CPU oracle --
def oracle_step(n, order, images, theta, ncrit):
    """One oracle FMM step (tree, traversal, evaluation) on TG n^3; returns
    (seconds, p2p pairs)."""
    import oracle
    import synth
    x, a, s = synth.taylor_green(n)
    t0 = time.perf_counter()
    f = oracle.OracleFMM(x, a, s, order=order, theta=theta, ncrit=ncrit, images=images)
    f.evaluate()
    dt = time.perf_counter() - t0
    cells = f.cells()
    p2p = f.p2p_list()
    pairs = int(np.sum(cells[p2p[:, 0], 5].astype(np.int64) * cells[p2p[:, 1], 5].astype(np.int64)))
    return dt, pairs


def cpu_baseline(args, theta):
    """SURVEY 8(d) CPU plan, on this host's cores (OpenMP, double): the oracle
    FMM timed on C1 and C2 (the metric's value is the C2 run, 174 x P2P pairs /
    s), and the direct sum's pair rate measured on a seeded target sample of
    C2 (free space), from which the full C1 periodic, C2 free-space and C3
    direct sums are extrapolated (labelled so; one pair = one evaluation of
    Eq. 1 + Eq. 3 per source image)."""
    import oracle
    import synth
    oracle.build()
    cores = os.cpu_count()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    out = {"unit": "TFLOP/s", "cores": int(os.environ["OMP_NUM_THREADS"]), "nproc": cores, "kind": "oracle"}
    # direct-sum pair rate: 4 x cores seeded targets of C2 against all 262,144 sources (free space)
    x, a, s = synth.taylor_green(64)
    nt = 4 * cores
    idx = np.random.default_rng(1106).choice(len(x), nt, replace=False)
    t0 = time.perf_counter()
    oracle.direct(x[idx], a[idx], x, a, s, images=0)
    dt = time.perf_counter() - t0
    rate = nt * len(x) / dt
    n1, n2, n3 = 16 ** 3, 64 ** 3, 256 ** 3
    img3 = 27 ** 3
    out["direct_pairs_per_s"] = rate
    out["direct_sample"] = "C2 free space, %d seeded targets x %d sources in %.2f s" % (nt, len(x), dt)
    out["c1_periodic_direct_s_extrapolated"] = n1 * n1 * img3 / rate
    out["c2_free_direct_s_extrapolated"] = n2 * n2 / rate
    out["c3_free_direct_s_extrapolated"] = n3 * n3 / rate
    out["c3_periodic_direct_s_extrapolated"] = n3 * n3 * img3 / rate
    fmm = {}
    for name, nside in (("c1", 16), ("c2", args.cpu_fmm_sample)):
        dtf, pairs = oracle_step(nside, args.order, args.images, theta, args.ncrit)
        fmm[name] = (dtf, pairs)
        out["%s_fmm_s" % name] = dtf
    dtf, pairs = fmm["c2"]
    out["value"] = FLOPS_PER_PAIR * pairs / dtf / 1e12
    out["sample"] = ("oracle FMM step (double, OpenMP, %d threads) on Taylor-Green %d^3 = %d particles (C2 at 64), "
                     "same p/theta/ncrit/k: %.2f s, %d P2P pairs; C1 FMM %.2f s; direct sums extrapolated from "
                     "the measured pair rate" % (out["cores"], args.cpu_fmm_sample, args.cpu_fmm_sample ** 3, dtf,
                                                 pairs, fmm["c1"][0]))
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    theta = theta_of(args.theta)
    cores = os.cpu_count()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    for _ in range(args.warmup):
        oracle_step(args.ref_sample, args.order, args.images, theta, args.ncrit)
    ts, pairs = [], 0
    for _ in range(args.steps):
        dt, pairs = oracle_step(args.ref_sample, args.order, args.images, theta, args.ncrit)
        ts.append(dt)
    tot = sum(ts)
    v = FLOPS_PER_PAIR * pairs * len(ts) / tot / 1e12
    sample = ("oracle FMM step (double, OpenMP) on Taylor-Green %d^3 = %d particles per step, p=%d, k=%d, "
              "theta=%s, ncrit=%d" % (args.ref_sample, args.ref_sample ** 3, args.order, args.images, args.theta,
                                      args.ncrit))
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(ts), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic Taylor-Green lattice",
        "config": {"workload": "C3 family (bounded CPU sample)", "sample": sample},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": int(os.environ["OMP_NUM_THREADS"]), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# -------------------------------------------------------------- our arm --
def load_profile_traffic():
    """dram bytes per P2P launch from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "latest_p2p.json")
    try:
        d = json.load(open(p))
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_1106_5273_b200 as P
    import synth

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    theta = theta_of(args.theta)

    # C3 at N = 1; the weak-scaling tiles (synth.taylor_green_tile, Z27) at N > 1
    tiled = world > 1 and args.mode == "tiled"
    tiles = synth.RANK_TILES[world] if tiled else (1, 1, 1)
    gen = {"tiled": synth.taylor_green_tile, "refined": synth.taylor_green_rank,
           "strong": synth.taylor_green_octants}[args.mode]
    balanced = world > 1 and args.partition == "orb"
    if balanced and args.mode != "strong":
        raise SystemExit("--partition orb needs --mode strong")
    if balanced:
        full = synth.taylor_green(args.side)
        x, a, s = (v[synth.scatter_to_ranks(len(full[0]), world, rank)] for v in full)
    elif world == 1 and args.workload == "jitter":
        x, a, s = synth.jittered_lattice(args.side, amp=1.0)
    else:
        x, a, s = gen(args.side, world, rank)
    if args.workload != "lattice" and world > 1:
        raise SystemExit("--workload variants are single-GPU")
    n = len(x)
    stream = torch.cuda.Stream()
    nccl_id = None
    if world > 1:
        obj = [P.fmm_comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    f = P.FMM(order=args.order, images=args.images, theta=theta, ncrit=args.ncrit, device=local,
              stream=stream.cuda_stream, nranks=world, rank=rank, nccl_id=nccl_id, tiles=tiles,
              partition=1 if balanced else 0)
    with torch.cuda.stream(stream):
        xd, ad, sd = (torch.from_numpy(v).cuda() for v in (x, a, s))
        ud = torch.empty((n, 3), device="cuda")
        dd = torch.empty((n, 3), device="cuda")
        if args.workload == "advected":
            # the state after one vortex-method step (NEXT-1): particles leave the lattice,
            # leaves gain/lose particles and the tree turns adaptive (the paper's lattice
            # only returns to uniform at reinitialisation)
            f.step(xd, ad, sd, 2.0 * float(s[0]), 0.0)
        torch.cuda.synchronize()
        x, a, s = (t.cpu().numpy() for t in (xd, ad, sd))

    def step():
        f.set_particles(xd, ad, sd)
        f.evaluate(ud, dd)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(max(3, args.warmup)):
            step()
    barrier()

    gpu_index = local
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES")
    if cvd:
        try:
            gpu_index = int(cvd.split(",")[local])
        except Exception:
            pass
    clk = ClockSampler(gpu_index)
    clk.start()
    time.sleep(0.3)
    # timed region: K steps, one CUDA event between consecutive steps (library stream)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with torch.cuda.stream(stream):
        evs[0].record(stream)
        for i in range(args.steps):
            step()
            evs[i + 1].record(stream)
    barrier()
    clocks = clk.stop()
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    ms_mean = evs[0].elapsed_time(evs[-1]) / args.steps
    ms = statistics.median(per_step)            # median of the timed steps
    # per-phase CUDA-event times and counters: separate untimed steps (no host work in the timed region)
    stats = []
    with torch.cuda.stream(stream):
        for _ in range(3):
            step()
            stats.append(f.stats())
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)

    pairs = stats[-1]["p2p_pairs"]
    launches = stats[-1]["launches"] * args.steps
    cub_calls = stats[-1]["cub_calls"] * args.steps
    phase = {k: statistics.median(st[k] for st in stats) for k in
             ("ms_keys", "ms_sort", "ms_tree", "ms_upward", "ms_traverse", "ms_m2l", "ms_m2l_tc", "ms_m2l_reg",
              "ms_p2p", "ms_downward", "ms_finalize", "ms_set_total", "ms_eval_total")}
    phase_ranks = [phase]
    if world > 1:
        phase_ranks = [None] * world
        mine = {k: round(v, 3) for k, v in phase.items()}
        mine.update({k: stats[-1][k] for k in ("n", "nleaves", "ncells_local", "ncells", "p2p_list", "p2p_pairs",
                                               "p2p_near_pairs", "m2l_list", "m2l_reg_list")})
        dist.all_gather_object(phase_ranks, mine)
    m2l_split = {k: stats[-1][k] for k in ("m2l_list", "m2l_tc_list", "m2l_reg_list")}
    m2l_split["tc_fraction"] = m2l_split["m2l_tc_list"] / max(1, m2l_split["m2l_list"])
    m2l_split["reg_kernel_tflops_algorithmic"] = (29040.0 * m2l_split["m2l_reg_list"] / (phase["ms_m2l_reg"] * 1e-3) / 1e12
                                                  if phase["ms_m2l_reg"] > 0 else None)
    m2l_split["reg_kernel_frac_fp32_peak"] = (m2l_split["reg_kernel_tflops_algorithmic"] / FP32_PEAK_TFLOPS
                                              if m2l_split["reg_kernel_tflops_algorithmic"] else None)

    # e2e through the C ABI from pinned host buffers
    e2e = None
    if not args.no_e2e:
        xh, ah, sh = (torch.from_numpy(v).pin_memory() for v in (x, a, s))
        uh = torch.empty((n, 3)).pin_memory()
        dh = torch.empty((n, 3)).pin_memory()
        ke = max(3, args.steps // 2)
        with torch.cuda.stream(stream):
            f.set_particles(xh, ah, sh)
            f.evaluate(uh, dh)
        barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(ke):
                f.set_particles(xh, ah, sh)
                f.evaluate(uh, dh)
            e1.record(stream)
        barrier()
        wall = (time.perf_counter() - t0) / ke
        ms_e2e = max(e0.elapsed_time(e1) / ke, 1e3 * wall)
        e2e = {"ms_per_step": ms_e2e, "h2d_bytes_per_step": int(xh.numel() * 4 + ah.numel() * 4 + sh.numel() * 4),
               "d2h_bytes_per_step": int(uh.numel() * 4 + dh.numel() * 4), "pairs": pairs}

    # aggregate over ranks: max time, summed work
    t = torch.tensor([ms, e2e["ms_per_step"] if e2e else 0.0, phase["ms_p2p"], ms_mean], dtype=torch.float64,
                     device="cuda")
    w = torch.tensor([float(pairs), float(n)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(w, op=dist.ReduceOp.SUM)
    ms_max, ms_e2e_max, p2p_ms_max, ms_mean_max = t.tolist()
    tot_pairs, tot_n = w.tolist()
    value = FLOPS_PER_PAIR * tot_pairs / (ms_max * 1e-3) / 1e12

    if rank == 0:
        traffic, prof = load_profile_traffic()
        from tools.sass_flops import p2p_flops_per_pair, sass_digest
        fpp = p2p_flops_per_pair(P.fmm.LIB_PATH)
        near = stats[-1]["p2p_near_pairs"]
        hw_flops = near * fpp.get("near", 0.0) + (pairs - near) * fpp.get("far", 0.0)
        flops_src = "static SASS count (tools/sass_flops.py)"
        # prefer the ncu-counted flops of this exact build on this exact workload
        if prof and prof.get("hw_flops_ncu") and prof.get("hw_flops_ncu_pairs") == pairs and \
                prof.get("sass_sha1") == sass_digest(P.fmm.LIB_PATH):
            hw_flops = prof["hw_flops_ncu"]
            flops_src = "ncu sm__sass_thread_inst_executed_op_{fadd,fmul,ffma,fadd2,fmul2,ffma2}_pred_on " \
                        "(same SASS, same workload; profiles/latest_p2p.json)"
        t_p2p = phase["ms_p2p"] * 1e-3
        achieved = hw_flops / t_p2p / 1e12
        roof = {"kernel": "k_p2p (near field, a12)", "bound": "alu", "achieved": achieved,
                "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / FP32_PEAK_TFLOPS,
                "traffic": traffic,
                "per_launch": {"ms": phase["ms_p2p"], "pairs": pairs, "near_pairs": int(near),
                               "hw_flops_per_pair_static": fpp, "hw_flops": hw_flops,
                               "hw_flops_per_pair": hw_flops / pairs if pairs else None, "hw_flops_source": flops_src},
                "model": {"flops_per_pair": FLOPS_PER_PAIR,
                          "achieved_tflops": FLOPS_PER_PAIR * pairs / t_p2p / 1e12,
                          "note": "paper-style Table 1 count (sqrt/rsqrt/exp/div = 1 flop); not a hardware rate"},
                "note": "achieved = hardware FP32 flops of one P2P launch (FADD/FMUL 1, FFMA 2, packed FP32x2 "
                        "ops per lane; source in per_launch.hw_flops_source) / "
                        "mean P2P launch time (CUDA events on the launch stream); peak = 148 SM x 128 FP32 lanes "
                        "x 2 x 1.965 GHz (derived, DESIGN.md; FFMA/FFMA2 probe measured 72.4/73.9 TFLOP/s)"}
        if prof:
            roof["profile"] = {k: prof[k] for k in prof if k != "dram_bytes_per_launch"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline(args, theta)
            except Exception as ex:  # the baseline never blocks the GPU number
                cpu = {"value": None, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "oracle",
                       "sample": "failed: %s" % ex}
        out = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max, "s_per_step": ms_max / 1e3,
            "timing": {"statistic": "median of the %d timed steps (CUDA events between steps, library stream; "
                                    "max over ranks)" % args.steps,
                       "ms_per_step_mean": ms_mean_max, "ms_steps_rank0": per_step},
            "higher_is_better": True, "scaling": "strong" if (world > 1 and args.mode == "strong") else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic Taylor-Green lattice (reading Z26), generated on host, resident in HBM",
            "config": {"workload": ("C3: Taylor-Green %d^3 = %d particles per GPU%s, periodic k=%d, p=%d, theta=%s, "
                                    "ncrit=%d" % (args.side, n, {"lattice": "", "jitter": " (stress: lattice jittered "
                                                                 "by +-h/4, seed 5273)",
                                                                 "advected": " (stress: after one fmm_step, midpoint "
                                                                 "RK2 with dt = h/2)"}[args.workload],
                                                  args.images, args.order, args.theta, args.ncrit))
                       if world == 1 else
                       ("C5 weak scaling: %s tiles of the 2pi Taylor-Green cube, one %d^3 = %d-particle tile per "
                        "GPU, periodic k=%d, p=%d, theta=%s, ncrit=%d (reading Z27)" %
                        ("x".join(str(m) for m in tiles), args.side, n, args.images, args.order, args.theta,
                         args.ncrit)) if tiled else
                       ("C4-style refinement: Taylor-Green lattice %s in [-pi,pi)^3, %d particles per GPU, "
                        "periodic k=%d, p=%d, theta=%s, ncrit=%d" %
                        ("x".join(str(args.side * m) for m in synth.RANK_LATTICE[world]), n,
                         args.images, args.order, args.theta, args.ncrit)) if args.mode == "refined" else
                       ("C4 strong scaling: Taylor-Green %d^3 in [-pi,pi)^3 %s, %d particles on "
                        "this GPU, periodic k=%d, p=%d, theta=%s, ncrit=%d" %
                        (args.side, "passed as random 1/N subsets and redistributed by the library every step "
                         "(ORB recursive multisection, partition = 1)" if balanced else
                         "split by Morton octants", n, args.images, args.order, args.theta, args.ncrit)),
                       "particles_total": int(tot_n), "step": "fmm_set_particles + fmm_evaluate (all 8a rows)",
                       "l2": "inputs larger than L2 (%.0f MB vs 126 MB); no flush" % (n * 28 / 1e6),
                       "parallelism": "1 GPU" if world == 1 else
                       "%d GPUs: %s domain decomposition, local trees + LET-MAC local essential trees "
                       "(cells, multipoles, bodies) over NCCL grouped send/recv on a comm stream overlapped "
                       "with the local near field, top multipoles all-reduced" %
                       (world, "ORB multisection (partition = 1)" if balanced else "Morton-octant / tile")},
            "let": None if world == 1 else {k: statistics.mean(st[k] for st in stats) for k in
                                            ("let_bytes_sent", "let_bytes_recv", "let_cells", "let_leaves", "ms_let",
                                             "ms_let_exposed", "let_fallback", "redist_bytes", "ncells",
                                             "ncells_local")},
            "p2p_pairs_per_step": int(tot_pairs), "model_flops_per_step": FLOPS_PER_PAIR * tot_pairs,
            "particles_per_s": tot_n / (ms_max * 1e-3),
            "phases_ms": phase,
            "phases_ms_per_rank": phase_ranks if world > 1 else None,
            "m2l_split": m2l_split,
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": None if not e2e else {
                "value": FLOPS_PER_PAIR * tot_pairs / (ms_e2e_max * 1e-3) / 1e12, "unit": "TFLOP/s",
                "ms_per_step": ms_e2e_max, "h2d_bytes_per_step": e2e["h2d_bytes_per_step"],
                "d2h_bytes_per_step": e2e["d2h_bytes_per_step"]},
            "gpu_launches": int(launches), "cub_calls": int(cub_calls),
            "clocks": clocks,
        }
        print(json.dumps(out), flush=True)
    f.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
