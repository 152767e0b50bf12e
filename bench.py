"""bench.py -- LDSolver rollout-step throughput on B200 (driver contract).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ldsolver|reference]
                [--config c4] [--precision tf32|fp32|f16|bf16] [--dry-run]

A "step" is one full LDSolver time step (all RK stages: conv net, fused stencil/
flux/RK kernel, FFT projection) over the config's batch of synthetic fields.
N GPUs run as N ranks, each owning its own batch (ensemble sharding, SURVEY.md
§8e PAR-1: no data-path collective, "scaling": "weak").  `--gpus N` without a
torchrun environment re-launches this script under torch.distributed.run with N
processes (127.0.0.1 rendezvous); under torchrun WORLD_SIZE must equal N.

Default workload: BASELINE.json configs[3] (c4: double shear layer 256^2, B=64 per
GPU, SSP-RK3 + FFT projection, 6x64 GELU net + TC head, TF32 conv) -- the largest
BASELINE config that fits one GPU unsplit (BASELINE's metric names no config;
VERDICT r01).  c2 (64^2, B=32: launch / L2-bound) is reported as a `variants`
entry in steps/s.

Metric: cell-updates/s = (ranks x B x N^2 x K) / max-over-ranks device time.
L2 is flushed (a 256 MiB write) between timed steps; each step is timed by its
own CUDA-event pair on the launching stream and the K durations are summed.
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

METRIC = "cell-updates/sec per LDSolver step"
UNIT = "cell-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None, help="ranks (GPUs); > 1 outside torchrun re-launches under "
                    "torch.distributed.run")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ldsolver", choices=["ldsolver", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--precision", default=None, choices=["tf32", "fp32", "f16", "bf16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip timing the other conv precisions and c2")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-elements", type=int, default=0,
                    help="batch elements in the CPU oracle sample (0: one per host core, at most B)")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo check of the multi-rank plumbing (no GPU)")
    ap.add_argument("--slab", action="store_true",
                    help="slab decomposition of ONE global problem over the ranks (NCCL halo exchange + "
                         "distributed FFT; SURVEY.md §8e PAR-2/3): strong scaling, e.g. --config c5a")
    ap.add_argument("--override", default="", help="measurement only: comma list k=v of config fields "
                    "(e.g. activation=0,batch=128); the JSON config records it")
    return ap.parse_args()


def workload(cfg):
    desc = {"c1": "2-D viscous Burgers", "c2": "2-D decaying incompressible NS",
            "c3": "2-D Kolmogorov forced flow", "c4": "2-D double shear layer",
            "c5a": "Kolmogorov turbulence", "c5b": "Kolmogorov turbulence ensemble"}[cfg.name]
    rk = {2: "RK2", 3: "SSP-RK3", 4: "RK4"}[cfg.rk_order]
    return (f"{cfg.name}: {desc} {cfg.n}x{cfg.n}, B={cfg.batch}/GPU, {rk}"
            f"{' + FFT projection' if cfg.system == 1 else ''}, {cfg.n_layers}x{cfg.width} "
            f"{'GELU' if cfg.activation == 1 else 'ReLU'} conv net{' + TC head' if cfg.tc_head else ''}")


# ------------------------------------------------------------------ clocks


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        if not self.rows:
            return None
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ CPU oracle baseline


def run_cpu_oracle(cfg, params, u0, seconds: float, elements: int = 0):
    """Time the plain C++ oracle (oracle/cpp, fp64, std::thread; north_star's "plain, slow CPU C++
    implementation") as it stands on a bounded sample of the workload: whole steps of the first
    `elements` batch elements (default 1: every host thread on the rows of that element) until
    `seconds` of wall time have elapsed (at least one step).  Elements are independent, so the
    throughput is reported per cell.  Returns (cell-updates/s, sample, cores, kind)."""
    from oracle import cpp_oracle as X
    k = max(1, min(elements or 1, cfg.batch))
    u = u0[:k].astype(np.float64)
    cores = X.hardware_threads()
    steps = 0
    t0 = time.perf_counter()
    while True:
        u = X.step(u, cfg, params, step_index=steps)
        steps += 1
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return (k * cfg.n * cfg.n * steps / el,
            f"{steps} C++-oracle step(s) of batch element(s) 0..{k - 1} ({cfg.n}x{cfg.n}) in {el:.1f} s "
            f"on {cores} threads",
            cores, "oracle (plain C++ fp64, std::thread; oracle/cpp/ldsolver_oracle.cpp)")


# ------------------------------------------------------------------ multi-process launch


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(a) -> None:
    """`--gpus N` (N > 1) outside torchrun: re-run this script as N ranks under
    torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous) and exit with its code.
    Under torchrun, WORLD_SIZE must equal --gpus (a mismatch would report the wrong n_gpus)."""
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None:
        if a.gpus is not None and a.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
                   "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
                   *sys.argv[1:]]
            sys.stdout.flush()
            r = subprocess.run(cmd)
            sys.exit(r.returncode)
        return
    if a.gpus is not None and int(world_env) != a.gpus and a.impl != "reference":
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world_env}\n")
        sys.exit(2)


def dry_run(a, rank, world):
    """CPU check of the multi-rank plumbing (gloo): the same rank / barrier / max-over-ranks /
    aggregation path as the GPU arm, with a host-side stand-in for the device time."""
    from paper_2507_01975_b200 import ensemble as E
    from ldgen.configs import get_config
    pg = E.init_process_group("gloo")
    cfg = get_config(a.config)
    cells = cfg.batch * cfg.n * cfg.n
    t0 = time.perf_counter()
    x = np.zeros(1 << 16)
    for _ in range(max(a.steps, 1)):
        x += 1.0
    ms = (time.perf_counter() - t0) * 1e3 + 1e-6
    ms_max = E.max_over_ranks(ms, pg)
    ranks = [rank]
    if pg:
        import torch.distributed as dist
        ranks = [None] * world
        dist.all_gather_object(ranks, rank)
        pg.barrier()
    if rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": E.aggregate_throughput(world, cells, a.steps, ms_max),
                          "unit": UNIT, "n_gpus": world, "ranks": ranks, "steps": a.steps, "warmup": a.warmup,
                          "config": {"workload": workload(cfg), "parallelism": f"ensemble x{world} (no collective)"}}))
    if pg:
        pg.destroy_process_group()


# ------------------------------------------------------------------ timing helpers


def time_steps(solver, u, stream, steps, flush, pg, dev):
    """K steps, each bracketed by its own CUDA-event pair on the launching stream, L2 flushed
    (outside the events) before each; barrier + synchronize on both sides; max over ranks."""
    import torch
    from paper_2507_01975_b200 import ensemble as E
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    if pg:
        pg.barrier()
    torch.cuda.synchronize(dev)
    for k in range(steps):
        flush.fill_(float(k))
        evs[k][0].record(stream)
        solver.ld_step(u, stream)
        evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    if pg:
        pg.barrier()
    ms = sum(s.elapsed_time(e) for s, e in evs)
    return E.max_over_ranks(ms, pg, dev)


def build_inputs(cfg, rank, world, slab=False):
    from ldgen import make_weights
    from ldgen.ic import make_config_ic
    from paper_2507_01975_b200.ensemble import shard
    if slab:   # every rank holds rows [r n, (r+1) n) of the same B fields
        ug = make_config_ic(cfg).astype(np.float32)
        cfg = cfg.with_dt(ug)
        nrow = cfg.n // world
        u0 = np.ascontiguousarray(ug[:, :, rank * nrow:(rank + 1) * nrow])
    else:
        u0 = make_config_ic(cfg, elements=shard(rank, world, cfg.batch)).astype(np.float32)
        cfg = cfg.with_dt(u0) if cfg.ic != "fourier" else cfg.with_dt(make_config_ic(cfg))
    params = make_weights(cfg.n_layers, cfg.width, cfg.n_out, seed=0, init="normal")
    if getattr(cfg, "fno_layers", 0) > 0:   # NEXT-2 branch: its blob follows the conv parameters
        from ldgen.spectral import spectral_blob
        params = np.concatenate([params, spectral_blob(cfg.fno_kmax, cfg.fno_width, cfg.fno_layers, seed=1,
                                                       scale=0.05)])
    if getattr(cfg, "tc_mode", 0) == 1:     # NEXT-3 history block: its blob comes last
        from ldgen.spectral import spectral_blob
        params = np.concatenate([params, spectral_blob(cfg.tc_kmax, cfg.tc_width, cfg.tc_layers, seed=2, scale=0.05,
                                                       n_in=2 * cfg.tc_interval, n_out=2)])
    return cfg, u0, params


PRECS = {"fp32": 0, "tf32": 1, "f16": 2, "bf16": 3}


def main():
    a = parse()
    self_launch(a)
    from paper_2507_01975_b200.ensemble import dist_env
    rank, world, local = dist_env()
    if a.dry_run:
        return dry_run(a, rank, world)
    from ldgen.configs import get_config

    cfg = get_config(a.config)
    prec = a.precision or "tf32"
    cfg = cfg.replace(conv_precision=PRECS[prec])
    if cfg.name == "c5b" and not (a.override and "batch=" in a.override):
        cfg = cfg.replace(batch=cfg.batch // 8)   # BASELINE c5b: batch 512 sharded over 8 GPUs -> 64 per GPU
    if a.override:
        cfg = cfg.replace(**{k: type(getattr(cfg, k))(v) for k, v in (kv.split("=") for kv in a.override.split(","))})
    B = cfg.batch

    if a.impl == "reference":
        # the reference arm of this tier is the CPU oracle (oracle/), on rank 0 only
        if rank != 0:
            return
        cfg, u0, params = build_inputs(cfg, 0, 1)
        cells = B * cfg.n * cfg.n
        vals, sample, cores, kind = [], "", 1, ""
        for _ in range(a.warmup):
            run_cpu_oracle(cfg, params, u0, 0.0, a.cpu_elements)
        for _ in range(a.steps):
            v1, sample, cores, kind = run_cpu_oracle(cfg, params, u0, 0.0, a.cpu_elements)
            vals.append(v1)
        v = statistics.median(vals)
        out = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus or world,
               "steps": a.steps, "warmup": a.warmup, "ms_per_step": cells / v * 1e3 if v else None,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (seeded IC + seeded random-init weights)",
               "config": {"workload": workload(cfg), "n": cfg.n, "batch_per_gpu": B},
               "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                                "sample": f"per step: {sample}; value = median over {a.steps} samples, "
                                          "scaled per cell (B elements are independent)"},
               "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return

    import torch
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2507_01975_b200 import ensemble as E
    from paper_2507_01975_b200 import ldsolver as L
    pg = E.init_process_group("nccl", device=dev)
    cfg, u0, params = build_inputs(cfg, rank, world, a.slab)
    cells = B * cfg.n * cfg.n // (world if a.slab else 1)   # cells this rank updates per step

    c = L.make_config(cfg)
    comm = None
    if a.slab:   # NCCL communicator of the library: id from rank 0, broadcast over torch.distributed
        uid = L.nccl_unique_id() if rank == 0 else bytes(128)
        if pg:
            t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
            pg.broadcast(t, 0)
            uid = bytes(t.cpu().tolist())
        comm = L.nccl_comm_init(uid, world, rank)
        dist_desc = L.ld_dist(mode=2, rank=rank, world=world, nccl_comm=comm)
    else:
        dist_desc = L.ld_dist(mode=1 if world > 1 else 0, rank=rank, world=world, nccl_comm=None)
    solver = L.Solver(c, params, dist=dist_desc, device=dev)
    stream = torch.cuda.current_stream(dev)
    u = torch.from_numpy(u0).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    for _ in range(max(a.warmup, 0)):
        solver.ld_step(u, stream)
    torch.cuda.synchronize(dev)

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ms_max = time_steps(solver, u, stream, a.steps, flush, pg, dev)
    clk = clocks.stop()
    value = E.aggregate_throughput(world, cells, a.steps, ms_max)
    if not os.environ.get("LD_XN_DEBUG"):   # measurement knobs produce garbage on purpose
        assert torch.isfinite(u).all(), "non-finite field in the timed run"

    # ---- per-kernel timing pass (same workload, same stream, events around each launch)
    solver.set_kernel_timing(True)
    for k in range(a.steps):
        flush.fill_(float(k))
        solver.ld_step(u, stream)
    kt = solver.kernel_times()
    solver.set_kernel_timing(False)

    # ---- end-to-end through the public host API (pinned host field, H2D + step + D2H per step)
    uh = torch.from_numpy(u0.copy()).pin_memory()
    e_ms = 0.0
    solver.ld_rollout_host(uh, 1, stream)   # warm the path
    for k in range(a.steps):
        flush.fill_(float(k))
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        solver.ld_rollout_host(uh, 1, stream)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms += ev0.elapsed_time(ev1)
    e2e_value = E.aggregate_throughput(world, cells, a.steps, E.max_over_ranks(e_ms, pg, dev))

    # ---- context: the other conv precisions on the same workload, and c2 (launch / L2-bound)
    variants = {}
    if not a.no_variants and not a.slab:
        vlist = [(vp, cfg) for vp in ("tf32", "f16", "bf16", "fp32") if vp != prec]
        if cfg.name != "c2" and not a.override:
            vlist.append(("c2_tf32", get_config("c2", conv_precision=1)))
        for name, vcfg in vlist:
            if name in PRECS:
                vcfg = vcfg.replace(conv_precision=PRECS[name])
                vu0, vparams = u0, params
            else:
                vcfg, vu0, vparams = build_inputs(vcfg, rank, world)
            sv = L.Solver(L.make_config(vcfg), vparams, dist=dist_desc, device=dev)
            uv = torch.from_numpy(vu0).to(dev)
            nv = max(3, a.steps // 4) if name == "fp32" else a.steps
            for _ in range(max(a.warmup, 3)):
                sv.ld_step(uv, stream)
            torch.cuda.synchronize(dev)
            vms = time_steps(sv, uv, stream, nv, flush, pg, dev)
            vcells = vcfg.batch * vcfg.n * vcfg.n
            variants[name] = {"value": E.aggregate_throughput(world, vcells, nv, vms), "ms_per_step": vms / nv,
                              "steps_per_s": 1e3 * nv / vms, "steps": nv,
                              "workload": workload(vcfg) + f", {['fp32', 'tf32', 'f16', 'bf16'][vcfg.conv_precision]} conv"}
            sv.close()
            del sv, uv
        # NEXT-4: the adjoint step (ld_step_vjp, fp32 SIMT) on c2 -- a training step's reverse pass
        vcfg, vu0, vparams = build_inputs(get_config("c2", conv_precision=0), rank, world)
        sv = L.Solver(L.make_config(vcfg), vparams, dist=dist_desc, device=dev)
        uv = torch.from_numpy(vu0).to(dev)
        gv = torch.ones_like(uv)
        gin = torch.empty_like(uv)
        gp = torch.zeros(vparams.size, device=dev)
        for _ in range(2):
            sv.ld_step_vjp(uv, gv, gin, gp, stream)
        torch.cuda.synchronize(dev)
        nv = max(3, a.steps // 4)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nv)]
        for k in range(nv):
            flush.fill_(float(k))
            evs[k][0].record(stream)
            sv.ld_step_vjp(uv, gv, gin, gp, stream)
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
        vms = E.max_over_ranks(sum(x.elapsed_time(y) for x, y in evs), pg, dev)
        vcells = vcfg.batch * vcfg.n * vcfg.n
        # FLOPs of one VJP: the net forward for the p-1 recomputed stage fields, and per
        # stage the net forward again plus its weight- and input-gradient convolutions (3 net-equivalents)
        chans = [2] + [vcfg.width] * (vcfg.n_layers - 1) + [vcfg.n_out]
        net_flop = sum(2 * 9 * a * b for a, b in zip(chans[:-1], chans[1:]))
        vflop = vcells * net_flop * ((vcfg.rk_order - 1) + 3 * vcfg.rk_order)
        mhz = 1965.0
        try:
            mhz = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("sm_max_mhz", mhz)
        except Exception:
            pass
        alu_peak = 148 * 128 * 2 * mhz * 1e6
        variants["vjp_c2"] = {"value": E.aggregate_throughput(world, vcells, nv, vms), "ms_per_call": vms / nv,
                              "steps": nv, "workload": workload(vcfg) + ", ld_step_vjp (u_bar and theta_bar), fp32 SIMT",
                              "roofline": {"bound": "alu", "achieved": vflop / (vms / nv * 1e-3) / 1e12,
                                           "peak": alu_peak / 1e12, "unit": "TFLOP/s",
                                           "frac": vflop / (vms / nv * 1e-3) / alu_peak,
                                           "algorithmic": f"{vflop:.4g} FLOP per call (net-equivalents: "
                                                          f"{(vcfg.rk_order - 1) + 3 * vcfg.rk_order})"}}
        sv.close()
        del sv, uv, gv, gin, gp

    if rank != 0:
        solver.close()
        if comm is not None:
            L.nccl_comm_destroy(comm)
        if pg:
            pg.destroy_process_group()
        return

    roof, shares = roofline(cfg, prec, kt, ms_max / a.steps, a.steps)
    cpu = None
    if not a.no_cpu_baseline:
        v, sample, cores, kind = run_cpu_oracle(cfg, params, u0, a.cpu_seconds, a.cpu_elements)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample}

    step_ms = ms_max / a.steps
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": step_ms, "steps_per_s": 1e3 / step_ms, "higher_is_better": True,
        "scaling": "strong" if a.slab else "weak",
        "vs_baseline": None, "dtype": {"tf32": "tf32", "f16": "f16 conv operands, f32 accumulate/stencil/FFT",
                                         "bf16": "bf16 conv operands, f32 accumulate/stencil/FFT", "fp32": "f32"}[prec],
        "data": "synthetic (seeded IC per BASELINE config + seeded random-init weights)",
        "config": {"workload": workload(cfg), "override": a.override or None, "n": cfg.n,
                   "batch_per_gpu": B if not a.slab else f"{B} (rows 1/{world} each)",
                   "global_batch": B if a.slab else B * world,
                   "dt": cfg.dt, "conv_precision": prec,
                   "parallelism": (f"slab x{world} (NCCL halos + distributed-FFT all-to-alls)" if a.slab
                                   else f"ensemble x{world} (no collective)"),
                   "l2": "flushed between timed steps (256 MiB write, outside the per-step events)"},
        "roofline": roof,
        "kernels": shares,
        "variants": variants,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(u0.nbytes),
                "d2h_bytes_per_step": int(u0.nbytes)},
        "gpu_launches": solver.launches_per_step() * a.steps,
        "clocks": clk,
    }
    print(json.dumps(out))
    solver.close()
    if comm is not None:
        L.nccl_comm_destroy(comm)
    if pg:
        pg.destroy_process_group()


# memory-bound classes: algorithmic bytes per cell per launch (DESIGN.md §6 / SURVEY.md §8d):
# fused flux/RK 120 B/cell-stage; projection 16 B/cell on chip (N <= 128: read U*, write U);
# N = 128..1024 real-data passes 40 B/cell (rows: U* 8 in, half spectrum 4 out; columns 4 + 4; inverse rows
# fused with the correction: spectrum 4 + U* 8 in, U 8 out -- p stays on chip; 48 with LD_PROJ_UNFUSED=1,
# which adds p 4 out + 4 in); N >= 2048 complex passes 64 B/cell
def flux_epilogue(cfg):
    """ldsolver.cu use_flux_epi: the tcgen05 output layer writes face fluxes (16 B/cell) instead of the 24
    stencils, and the flux class is flux_div_kernel (F 16 + U 8 + u^n 8 read, 8 written per cell-stage)."""
    return (os.environ.get("LD_FLUX_EPI", "1") != "0" and cfg.conv_precision != 0 and cfg.stencil_mode == 0
            and not getattr(cfg, "freeze_stencils", 0) and getattr(cfg, "fno_layers", 0) == 0
            and cfg.n >= 128 and cfg.n % 128 == 0)


def mem_bytes_per_cell(name, n, batch=1, fepi=False):
    cluster = n < 128   # fft.cu projection_uses_pencil
    r2 = 48.0 if os.environ.get("LD_PROJ_UNFUSED") else 40.0
    proj = 16.0 if cluster else (r2 if n <= 1024 else 64.0)
    return {"flux_rk": 40.0 if fepi else 120.0, "projection": proj, "flux_proj": 120.0}.get(name)


def roofline(cfg, prec, kt, step_ms, steps):
    """Roofline object of the dominant kernel class + per-class shares of the step."""
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    B, W, N2 = cfg.batch, cfg.width, cfg.n * cfg.n
    dom = max(kt, key=lambda k: kt[k][0])
    dom_ms, dom_n = kt[dom]
    per_launch_s = dom_ms / max(dom_n, 1) * 1e-3
    traffic = None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        traffic = prof.get(cfg.name, {}).get(prec, {}).get(dom)
    except Exception:
        pass
    if dom.startswith("conv"):
        ci = 2 if dom == "conv_first" else W
        co = cfg.n_out if dom == "conv_last" else W
        # the net runs in L2-sized sub-batches: FLOPs per launch = the class's FLOPs per
        # step / its launches per step
        full = (cfg.n_layers - 2) * cfg.rk_order if dom == "conv_hidden" else cfg.rk_order
        chunks = max(1.0, (dom_n / steps) / full)
        flops = 2.0 * B * N2 * 9 * ci * co / chunks
        ach = flops / per_launch_s / 1e12
        frac_burst = None
        if prec in ("tf32", "f16", "bf16") and dom != "conv_first":
            # B200_PROFILING.md: the burst GEMM figure is the denominator for a kernel timed alone, the
            # sustained one (seconds-long loop under the power cap) for a kernel timed inside a long
            # step -- this kernel is timed over K back-to-back steps, so the sustained figure is the
            # denominator; the burst fraction is reported beside it
            ratio = 0.5 if prec == "tf32" else 1.0
            burst = peaks.get("bf16_tflops", 1590.0) * ratio
            sustained = peaks.get("bf16_tflops_sustained")
            peak, bound = (sustained * ratio if sustained else burst), "tensor"
            frac_burst = ach / burst
            src = (("measured" if "bf16_tflops" in peaks else "fallback") +
                   (" bf16_tflops_sustained" if sustained else " bf16_tflops (burst)") +
                   (" x 0.5 (nominal tf32/bf16 ratio)" if prec == "tf32" else " (f16 = bf16 rate)") +
                   "; kernel timed inside a long step")
        else:
            mhz = peaks.get("sm_max_mhz", 1965.0)
            peak, bound, src = 148 * 128 * 2 * mhz * 1e6 / 1e12, "alu", "148 SM x 128 FP32 FMA/clk x 2 x sm_max_mhz"
        roof = {"kernel": dom, "bound": bound, "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                "frac": ach / peak, "frac_vs_burst_peak": frac_burst, "traffic": traffic, "peak_source": src,
                "algorithmic": f"2*(B/{chunks:g})*N^2*9*{ci}*{co} = {flops:.4g} FLOP per launch ({chunks:g} sub-batches)",
                "algorithmic_bytes": (f"{B * N2 * (4 * ci + 24) / chunks:.4g} B per launch (read {4 * ci} + field 8, "
                                      "write face fluxes 16 B/cell: flux epilogue)"
                                      if dom == "conv_last" and flux_epilogue(cfg) else
                                      f"{B * N2 * 4 * (ci + co) / chunks:.4g} B per launch (read {4 * ci} + write {4 * co} B/cell)")}
    else:
        per_cell = mem_bytes_per_cell(dom, cfg.n, cfg.batch, flux_epilogue(cfg))
        byts = per_cell * B * N2
        ach = byts / per_launch_s / 1e9
        peak = peaks.get("hbm_gbs", 6650.0)
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": traffic, "peak_source": "measured hbm_gbs" if "hbm_gbs" in peaks else "fallback",
                "algorithmic": f"{per_cell} B/cell x {B * N2} cells per launch"}
    shares = {k: {"ms_per_launch": (v[0] / v[1] if v[1] else 0.0), "launches_per_step": v[1] / steps,
                  "share_of_step": v[0] / steps / step_ms if step_ms else 0.0} for k, v in kt.items() if v[1]}
    hbm = peaks.get("hbm_gbs", 6650.0)
    for k in shares:
        bpc = mem_bytes_per_cell(k, cfg.n, cfg.batch, flux_epilogue(cfg))
        if bpc and shares[k]["ms_per_launch"] > 0:
            gbs = bpc * B * N2 / (shares[k]["ms_per_launch"] * 1e-3) / 1e9
            shares[k].update({"algorithmic_bytes_per_cell": bpc, "achieved_gbs": gbs, "hbm_frac": gbs / hbm})
    return roof, shares


if __name__ == "__main__":
    main()
