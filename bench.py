#!/usr/bin/env python
"""bench.py -- fp64 transforms/s of the extra-component apply on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]

One "step" is one xc_apply of the whole hot path (SpMM on the FP64 tensor cores
over every block + dense tail, then the per-block inverse FFTs with the fused
W^{-1}/truncate epilogue) over one batch of B right-hand sides already resident
in HBM.  Default workload: BASELINE.json configs[4] (c5: Legendre N = 65536,
B = 4096 per GPU, eps = 1e-12; the config the metric's 1/2/4/8-GPU scaling is
quoted on).  Multi-GPU: one rank per GPU (torchrun; `--gpus N` without a
launcher re-launches itself under torch.distributed.run), the operator replicated
(built by the distributed precompute: node range per rank + NCCL all-gather) and
the config's seeded batch sharded by column with no collective on the data path
(strong scaling of the global B = 4096, the default; --weak gives every rank the
whole batch).

Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2004_11610_b200 import inputs as I  # noqa: E402

DMMA_PEAK_TFLOPS = 37.1   # measured: tools/fp64_peak.cu, mma.m8n8k4.f64 (profiles/fp64_peak_r01.txt)
DFMA_PEAK_TFLOPS = 33.9   # measured: same microbenchmark, DFMA


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class Clocks:
    """nvidia-smi clock/throttle sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, device):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={device}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def wait_ready(self, timeout=8.0):
        """Block until the sampler has written its first line (a cold nvidia-smi can take longer to
        start than a short timed region lasts)."""
        t0 = time.perf_counter()
        while self.p is not None and time.perf_counter() - t0 < timeout:
            if os.path.getsize(self.f.name) > 0:
                return
            time.sleep(0.05)

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _nodes(cfg, device):
    from paper_2004_11610_b200 import xc
    if cfg.kind == I.KIND_COS:
        return I.cos_nodes(cfg.N, cfg.seed), None
    if cfg.kind == I.KIND_EXP:
        return I.exp_nodes(cfg.N, cfg.seed), None
    if cfg.kind == I.KIND_LAGSPEC:
        return I.lagspec_freqs(cfg.N, cfg.T), None
    if cfg.kind == I.KIND_LAG2D:
        return I.lag2d_grid(cfg.N, cfg.eta), None
    x, w, wt = xc.gauss_rule(cfg.kind, cfg.N, cfg.alpha, cfg.beta, device=device)
    return x, wt


def _timing_nodes(cfg):
    """Nodes for the CPU timing legs only (the dense product's cost does not depend on node
    accuracy): scipy's Gauss rules (library routines), not the product."""
    import scipy.special
    if cfg.kind == I.KIND_COS:
        return I.cos_nodes(cfg.N, cfg.seed)
    if cfg.kind == I.KIND_EXP:
        return I.exp_nodes(cfg.N, cfg.seed)
    if cfg.kind == I.KIND_LAGSPEC:
        return I.lagspec_freqs(cfg.N, cfg.T)
    if cfg.kind == I.KIND_LAG2D:
        return I.lag2d_grid(cfg.N, cfg.eta)
    if cfg.kind == I.KIND_LAGUERRE:
        return np.linspace(0.0, 4.0 * cfg.N, cfg.N)   # scipy's Laguerre rule overflows at this N
    if cfg.N > 8192:
        # scipy's rules are an O(N^2) banded eigenvalue solve (minutes at N = 65536, which once ran
        # the reference arm into its time limit): the classical first-order estimate of the Gauss-
        # Jacobi nodes, theta_k = pi (2k + alpha - 1/2) / (2N + alpha + beta + 1), serves the timing
        k = np.arange(1, cfg.N + 1, dtype=np.float64)
        return np.sort(np.cos(np.pi * (2.0 * k + cfg.alpha - 0.5) / (2.0 * cfg.N + cfg.alpha + cfg.beta + 1.0)))
    if cfg.alpha == 0.0 and cfg.beta == 0.0:
        return scipy.special.roots_legendre(cfg.N)[0]
    return scipy.special.roots_jacobi(cfg.N, cfg.alpha, cfg.beta)[0]


CPU_COLS = 16   # the oracle's timed column count (the c5 check columns), fixed for both CPU legs


def _oracle_op_cached(cfg):
    """The oracle's c5 operator from tools/make_c5_oracle.py's cache (bands -> the oracle's sparse
    node-by-bin form), or None."""
    path = os.path.join(ROOT, "oracle_cache", "c5_oracle.npz")
    if cfg.name != I.CONFIGS["c5"].name or not os.path.exists(path):
        return None
    import scipy.sparse as sp

    import oracle as O
    z = np.load(path)
    kind = O.Kind(cfg.kind, cfg.alpha, cfg.beta)
    plan = O.make_plan(kind, cfg.N, cfg.eps)
    S = []
    for i, b in enumerate(plan.blocks):
        st, ln, v = z[f"start{i}"].astype(np.int64), z[f"len{i}"].astype(np.int64), z[f"vals{i}"]
        row = np.repeat(np.arange(cfg.N), ln)
        off = np.concatenate([[0], np.cumsum(ln)])
        col = st[row] + (np.arange(v.size) - off[row])
        S.append(sp.csr_matrix((v, (row, col)), shape=(cfg.N, b.H)))
    P = O.entries(kind, z["x"], 0, plan.tail).T.copy()
    return O.Operator(plan, S, [O.kaiser(plan.zeta, b.L - 1) for b in plan.blocks], P), z["x"]


def _dense_sample(cfg, threads):
    """The oracle's dense direct product (the paper's 'direct method'; entries regenerated in
    double-double) on CPU_COLS columns of the seeded batch and output rows [0, ndeg): (rate per full
    transform, seconds, ndeg, rows, nodes, X)."""
    import oracle as O
    os.environ["OMP_NUM_THREADS"] = str(threads)
    kind = O.Kind(cfg.kind, cfg.alpha, cfg.beta, eta=cfg.eta)
    x = _timing_nodes(cfg)
    X = I.config_rhs(cfg, B=CPU_COLS)
    cplx = cfg.kind in (I.KIND_EXP, I.KIND_LAGSPEC)
    rows_total = (cfg.M or cfg.N) if cplx else cfg.N
    ndeg = rows_total if (cplx or cfg.kind == I.KIND_LAG2D or cfg.N <= 16384) else 8192
    t0 = time.perf_counter()
    if cplx:
        O.dense_apply(kind, x, X, M=cfg.M or None)
    elif cfg.kind == I.KIND_LAG2D:   # the series sum D C = the transposed Laguerre product
        O.dense_apply_t(O.Kind(O.KIND_LAGUERRE), x, X)
    else:
        O.dense_apply_rows(kind, x, X, ndeg)
    t = time.perf_counter() - t0
    return CPU_COLS * (ndeg / rows_total) / t, t, ndeg, rows_total, x, X


def cpu_oracle_timing(cfg, threads, direction="A"):
    """The oracle as it stands, on CPU_COLS columns of the config's seeded batch, all host cores:
    (1) the dense direct product on output rows [0, ndeg) (_dense_sample; rate per full transform),
        with the double-double generation of the same entries timed alone beside it;
    (2) the oracle's compressed apply (Alg. 2 / Alg. 1 block form, library FFT) on the same
        columns, when its operator is at hand (built here for N <= 16384; c5 from the cache of
        tools/make_c5_oracle.py).
    Returns the cpu_baseline object; value = (1)."""
    import oracle as O
    kind = O.Kind(cfg.kind, cfg.alpha, cfg.beta, eta=cfg.eta)
    v, t_dense, ndeg, rows_total, x, X = _dense_sample(cfg, threads)
    cplx = cfg.kind in (I.KIND_EXP, I.KIND_LAGSPEC)
    t_gen = None
    if not cplx:   # the entry generation alone: the same rows x all nodes, node chunks of 4096
        gk = O.Kind(O.KIND_LAGUERRE) if cfg.kind == I.KIND_LAG2D else kind
        t0 = time.perf_counter()
        for k0 in range(0, cfg.N, 4096):
            O.entries(gk, x[k0:k0 + 4096], 0, ndeg)
        t_gen = time.perf_counter() - t0
    out = {"value": v, "unit": "transforms/s", "cores": threads, "kind": "oracle",
           "sample": f"dense direct product (double-double entries regenerated), {CPU_COLS} columns x "
                     f"output rows [0,{ndeg}) of {rows_total}: {t_dense:.2f} s; rate per full transform",
           "dense_s": t_dense, "entry_generation_s": t_gen, "columns": CPU_COLS, "rows": ndeg}
    comp = None
    try:
        op, t_build = None, None
        if cfg.kind != I.KIND_LAG2D and not cplx and cfg.N <= 16384:
            t0 = time.perf_counter()
            op = O.compress(O.make_plan(kind, cfg.N, cfg.eps, eps2=cfg.eps2), x)
            t_build = time.perf_counter() - t0
        elif cfg.kind != I.KIND_LAG2D and not cplx:
            got = _oracle_op_cached(cfg)
            if got is not None:
                op, _ = got
        if op is not None:
            n, t0 = 0, time.perf_counter()
            while True:
                if direction == "WAT":
                    O.apply_input_axis(op, X, np.ones(cfg.N))
                else:
                    O.apply_output_axis(op, X)
                n += 1
                if time.perf_counter() - t0 >= 2.0:
                    break
            t_ap = (time.perf_counter() - t0) / n
            comp = {"value": CPU_COLS / t_ap, "unit": "transforms/s", "seconds_per_apply": t_ap, "repeats": n,
                    "precompute_s": t_build,
                    "sample": f"oracle compressed apply ({'input' if direction == 'WAT' else 'output'} axis, "
                              f"library FFT) on the same {CPU_COLS} columns"}
    except Exception as e:  # pragma: no cover - reported, not fatal
        comp = {"error": repr(e)[:200]}
    out["compressed"] = comp
    return out


def run_reference(args, cfg, ws, rank):
    """--impl reference: the CPU oracle timed on the host cores (rank 0 only): per step the dense
    direct product on the fixed column sample, median over the timed steps; the first step also
    times the entry generation and the oracle's compressed apply (cpu_oracle_timing)."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    direction = args.direction or cfg.dirs[0]
    first = cpu_oracle_timing(cfg, threads, direction)
    vals = [first["value"]]
    for _ in range(args.warmup + args.steps - 1):
        vals.append(_dense_sample(cfg, threads)[0])
    v = float(np.median(vals[args.warmup:] if len(vals) > args.warmup else vals))
    base = dict(first)
    base["value"] = v
    line = {"impl": "reference", "metric": "fp64 transforms/s", "value": v, "unit": "transforms/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "N": cfg.N, "global_batch": cfg.B, "eps": cfg.eps,
                       "direction": direction},
            "cpu_baseline": base,
            "e2e": {"value": v, "unit": "transforms/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


COLL_DEVICE = "cuda"   # where the timing collectives' tensors live ("cpu" with the gloo test backend)


def sum_cols(B):
    from paper_2004_11610_b200.shard import sum_over_ranks
    return sum_over_ranks(B, device=COLL_DEVICE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=sorted(I.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--weak", action="store_true", help="every rank applies the whole batch (default: strong "
                    "scaling, the config's global batch sharded by column)")
    ap.add_argument("--batch", type=int, default=0, help="override the global batch (strong) / per-rank batch (weak)")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--direction", default="", help="A or WAT (default: the config's first)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group backend (gloo: host-mediated exchanges, for the 2-rank test on one GPU)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = I.CONFIGS[args.config]
    from paper_2004_11610_b200.shard import rank_columns, relaunch_cmd, world_from
    ws, rank, local, relaunch = world_from(os.environ, args.gpus)
    if relaunch:   # `bench.py --gpus N` without a launcher: one rank per GPU under torch.distributed.run
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")            # communicator lines (ranks, transport) on stderr
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        sys.exit(subprocess.call(relaunch_cmd(os.path.abspath(__file__), sys.argv[1:], args.gpus, port,
                                              sys.executable), env=env))

    if args.impl == "reference":
        run_reference(args, cfg, ws, rank)
        return

    import torch
    from paper_2004_11610_b200 import xc
    global COLL_DEVICE
    # XC_BENCH_ONE_DEVICE=1 (tests only): every rank on cuda:0 with the gloo backend -- the exchanges
    # and timing collectives then run on the host, no kernel waits on another rank
    if os.environ.get("XC_BENCH_ONE_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        # the NCCL communicator lines (ranks, devices, transport) on stderr, also under the driver's
        # own torchrun launch
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
            COLL_DEVICE = "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    direction = xc.XC_DIR_WAT if (args.direction or cfg.dirs[0]) == "WAT" else xc.XC_DIR_A
    B_global = args.batch or cfg.B
    cols = rank_columns(B_global, rank, ws, strong=not args.weak)
    B = cols.stop - cols.start
    # ---- precompute (not timed in the metric) ----
    t0 = time.perf_counter()
    x, wt = _nodes(cfg, local)
    t_nodes = time.perf_counter() - t0
    dirs = xc.XC_DIR_A | (xc.XC_DIR_WAT if "WAT" in cfg.dirs else 0)
    t0 = time.perf_counter()
    # N > 1: distributed precompute (node range per rank, NCCL all-gather of the node bands)
    T = xc.Transform(cfg.kind, x, cfg.eps, alpha=cfg.alpha, beta=cfg.beta, dirs=dirs, weights=wt, device=local,
                     dist=(rank, ws, xc.nccl_allgather() if args.dist_backend == "nccl" else xc.host_allgather())
                     if ws > 1 else None,
                     eta=cfg.eta, n_rows=cfg.M, eps2=cfg.eps2 if cfg.eps2 != 1e-2 else 0.0)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    info = T.info()

    # ---- inputs: seeded on the host, this rank's shard, resident in HBM ----
    from paper_2004_11610_b200.shard import max_over_ranks
    Xfull = I.config_rhs(cfg, B=B_global)   # the config's seeded batch; this rank's column shard
    if cfg.kind in (I.KIND_EXP, I.KIND_LAGSPEC):   # complex RHS, planar layout of the C ABI (2N rows)
        Xh = np.ascontiguousarray(np.concatenate([Xfull.real[:, cols], Xfull.imag[:, cols]]))
    else:
        Xh = np.ascontiguousarray(Xfull[:, cols])
    del Xfull
    X = torch.from_numpy(Xh).cuda()
    Y = torch.empty((T.rows(direction)[1], B), dtype=torch.float64, device=X.device)
    T.reserve(B)
    stream = torch.cuda.current_stream()

    torch.cuda.nvtx.range_push("xc_apply")
    for _ in range(args.warmup):
        T.apply(X, direction, out=Y)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = Clocks(local) if rank == 0 else None
    if clocks:
        clocks.wait_ready()
    # ---- timed region: xc_apply as a user calls it (its default CUDA-graph replay: a call
    # repeated with the same arguments is captured on its 2nd occurrence and replayed after) ----
    for _ in range(2):
        T.apply(X, direction, out=Y)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(args.steps):
        T.apply(X, direction, out=Y)
    ev1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    clk = clocks.stop() if clocks else None
    ms = max_over_ranks(ms, device=COLL_DEVICE)
    total_cols = int(round(sum_cols(B)))
    value = total_cols / (ms / 1e3)

    # ---- the same steps with per-phase CUDA events (profiling launches eagerly, no graph):
    # the dominant kernel's duration for the roofline ----
    T.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    p0.record(stream)
    for _ in range(args.steps):
        T.apply(X, direction, out=Y)
    p1.record(stream)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    prof = T.profile_read()
    T.profile(False)
    ems = max_over_ranks(p0.elapsed_time(p1) / args.steps, device=COLL_DEVICE)
    graph = {"eager_ms_per_step": ems, "eager_value": total_cols / (ems / 1e3), "unit": "transforms/s",
             "note": "value/ms_per_step: xc_apply's default CUDA-graph replay; eager: the same steps "
                     "launched kernel by kernel with per-phase events (the roofline's kernel times)"}

    # ---- roofline of the dominant kernel (SpMM on the FP64 tensor cores) ----
    nnz, tail, N = info["nnz"], info["tail"], info["N"]
    cmul = 8.0 if cfg.kind in (I.KIND_EXP, I.KIND_LAGSPEC, I.KIND_LAG2D) else 4.0   # complex x complex / x real
    spmm_flops = (cmul * nnz + 2.0 * tail * N) * B          # algorithmic, per launch
    spmm_ms = prof["ms_spmm"] / max(1, prof["n"])
    fft_ms = prof["ms_fft"] / max(1, prof["n"])
    if cfg.kind == I.KIND_LAG2D:   # no dense tail inside the product launch (separate kernels)
        spmm_flops = 8.0 * nnz * B
    achieved = spmm_flops / (spmm_ms / 1e3) / 1e12
    alg_bytes = info["alg_bytes_per_col"] * B + info["alg_bytes_fixed"]   # X in, Y out, operator once (SURVEY d.3)
    peaks = _peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # DRAM traffic of the SpMM launch from the committed ncu --set full capture (same workload)
    traffic, traffic_src = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "r02_spmm_traffic.json")))
        if tr.get("workload") == cfg.name and tr.get("B_per_gpu") == B and direction == xc.XC_DIR_A:
            traffic = float(tr["dram_bytes_read_per_launch"] + tr["dram_bytes_write_per_launch"])
            traffic_src = tr["source"]
    except Exception:
        traffic = None

    # ---- end to end: host buffers through xc_apply_host (copies inside the call) ----
    e2e = None
    if args.e2e_steps > 0:
        Xp = torch.from_numpy(Xh).pin_memory()
        Yp = torch.empty(tuple(Y.shape), dtype=torch.float64).pin_memory()
        T.apply_host_ptr(Xp.data_ptr(), Yp.data_ptr(), B, direction, stream=stream.cuda_stream)
        if dist:
            dist.barrier()
        # streaming host-buffer calls (xc_apply_host_async: consecutive calls overlap their copy
        # in / copy out), then one wait; wall clock on the host around the whole sequence
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        tw0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            T.apply_host_async_ptr(Xp.data_ptr(), Yp.data_ptr(), B, direction, stream=stream.cuda_stream)
        T.host_wait()
        ems = (time.perf_counter() - tw0) * 1e3 / args.e2e_steps
        ems = max_over_ranks(ems, device=COLL_DEVICE)
        e2e = {"value": total_cols / (ems / 1e3), "unit": "transforms/s",
               "h2d_bytes_per_step": int(sum_cols(Xh.nbytes)), "d2h_bytes_per_step": int(sum_cols(8 * Y.numel())),
               "ms_per_step": ems,
                   "api": "xc_apply_host_async x steps + xc_host_wait (pinned host buffers; host wall clock)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_timing(cfg, os.cpu_count() or 1, "WAT" if direction == xc.XC_DIR_WAT else "A")

    if rank == 0:
        line = {
            "metric": "fp64 transforms/s", "value": value, "unit": "transforms/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded N(0,1) RHS, Gauss nodes computed on the GPU)",
            "config": {"workload": cfg.name, "N": cfg.N, "B_per_gpu": B, "global_batch": total_cols,
                       "columns_of_rank0": [cols.start, cols.stop],
                       "eps": cfg.eps, "direction": "A" if direction == xc.XC_DIR_A else "WAT",
                       "parallelism": f"rhs-shard x{ws}, operator replicated",
                       "l2": "inputs larger than L2 (X = %.2f GB, partial sums %.2f GB)" % (
                           Xh.nbytes / 1e9, T.workspace_bytes(B) / 1e9),
                       "blocks": [b["L"] for b in T.blocks()], "tail": tail},
            "hbm_gbs": alg_bytes / (ms / 1e3) / 1e9,
            "hbm_frac": alg_bytes / (ms / 1e3) / 1e9 / hbm_peak,
            "fp64_tflops": info["flops_per_col_A"] * B / (ms / 1e3) / 1e12,
            "roofline": ({"bound": "tensor", "kernel": "bsr2d (8x4 complex blocks, mma.m8n8k4.f64)",
                          "achieved": achieved, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                          "frac": achieved / DMMA_PEAK_TFLOPS,
                          "peak_source": "measured DMMA microbenchmark (tools/fp64_peak.cu)"}
                         if cfg.kind == I.KIND_LAG2D else
                         {"bound": "tensor", "kernel": "spmm_dmma (mma.m8n8k4.f64)", "achieved": achieved,
                          "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": achieved / DMMA_PEAK_TFLOPS,
                          "peak_source": "measured DMMA microbenchmark (tools/fp64_peak.cu)"}) | {
                         "traffic": traffic, "traffic_unit": "bytes per launch", "traffic_source": traffic_src,
                         "spmm_ms": spmm_ms, "fft_ms": fft_ms, "spmm_share": spmm_ms / ms,
                         # the whole step against the fp64 roof: SURVEY 8d.3 flops (SpMM + tail + FFTs)
                         # per column x B / the measured DMMA peak / ms_per_step
                         "step_frac": info["flops_per_col_A" if direction == xc.XC_DIR_A else "flops_per_col_WAT"]
                                      * B / (DMMA_PEAK_TFLOPS * 1e12) / (ms / 1e3),
                         "dmma_issue_efficiency": (cmul * nnz + 2.0 * tail * N) / max(1.0, info["dmma_flops_per_col_A"])},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "graph": graph,
            "gpu_launches": T.launches(B, direction) * args.steps,   # xc_launches: kernels of one apply of B
            "clocks": clk,
            "comm": ({"backend": args.dist_backend, "world_size": ws,
                      "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                      "data_path_collectives": 0, "precompute": "2 all-gathers of node bands (xc_build_local/step)"}
                     if ws > 1 else None),
            "precompute_s": {"gauss_nodes": t_nodes, "build": t_build,
                             "mode": f"node range split over {ws} ranks + NCCL all-gather" if ws > 1 else "one GPU"},
            "nnz": nnz,
        }
        print(json.dumps(line), flush=True)
    T.close()
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
