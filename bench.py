#!/usr/bin/env python3
"""Benchmark of the dual-free grid-metric hot path on B200.

Metric (BASELINE.json): tets/s for lumped directed-area vectors + median-dual
volumes (fp64), and the fraction of the HBM roofline.  One "step" is one pass
of the SPEC timed region over the resident grid: the
dual-free element loop + boundary pass (one fused kernel) and the edge-based
volume loop, with the edge structures prebuilt.  Workload: BASELINE config 5
(256^3 Kuhn cube, 100,663,296 tets, +-0.15h jitter), the configuration the
metric is quoted on; seeded synthetic grid (SPEC meshgen, splitmix64 seed 42).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU: the path is single-GPU (north_star); N>1 runs N independent
replicas (one per rank, torchrun), whole-job tets/s = N*K*N_E / max-over-ranks
time ("scaling": "weak").
"""
from __future__ import annotations

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

METRIC = "tets/s for directed-area vectors + dual volumes (fp64); % of HBM roofline"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback, GB/s


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def algorithmic_bytes(mesh, n_edges, n_bnd_nodes, n_bnd_edges):
    """SURVEY.md 8(d) canonical bytes (each quantity counted once)."""
    D = mesh.dim
    L = D * (D + 1) // 2
    nE, nv, nB = mesh.num_elements(), mesh.num_nodes(), mesh.num_boundary()
    b_elem = 4 * (D + 1) * nE + 4 * L * nE + 8 * D * nv + 8 * D * n_edges
    b_bnd = 4 * D * nB + 8 * D * n_bnd_nodes + 16 * D * n_bnd_edges
    b_vol = 8 * n_edges + 8 * D * n_edges + 8 * D * nv + 8 * nv
    b_edges = (4 * (D + 1) * nE + 8 * n_edges + 8 * (nv + 1) + 4 * L * nE + 4 * L * nE
               + 4 * (n_edges + 1))
    return {"elem": b_elem, "bnd": b_bnd, "vol": b_vol, "metrics": b_elem + b_bnd + b_vol,
            "edges": b_edges}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def _rows(self):
        out = []
        try:
            lines = open(self.path).read().splitlines()
        except OSError:
            return out
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                t = time.mktime(time.strptime(parts[0].split(".")[0], "%Y/%m/%d %H:%M:%S"))
                t += float("0." + parts[0].split(".")[1]) if "." in parts[0] else 0.0
                out.append((t, float(parts[1]), float(parts[2]), parts[3:7]))
            except (ValueError, IndexError):
                continue
        return out

    def live(self) -> bool:
        """True once nvidia-smi has written samples (it starts slowly)."""
        return self.proc is not None and len(self._rows()) >= 2

    def stop(self, t0=None, t1=None):
        """Clock samples inside the host-time window [t0, t1] of the timed
        region (all samples if the window caught none)."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        self.proc.wait()
        rows = self._rows()
        os.unlink(self.path)
        inside = [r for r in rows if t0 is None or (t0 - 0.02 <= r[0] <= t1 + 0.02)]
        sel = inside or rows
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in sel:
            for nm, v in zip(names, r[3]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median([r[1] for r in sel])) if sel else None,
                "sm_max_mhz": max(r[2] for r in sel) if sel else None,
                "reasons": sorted(reasons), "samples": len(sel),
                "samples_in_timed_region": len(inside) if t0 is not None else None}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local, dist


def max_over_ranks(dist, value, device=None):
    if dist is None:
        return value
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# ---------------------------------------------------------------- CPU baseline
def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_rows(config, scale, steps, warmup, serial_reps, trad_reps, threads=None):
    """The reference CPU path on the bench's own workload (SPEC time_algorithms,
    SPEC.md:382-390,414): the oracle (oracle/oracle.c, CPU restatement of the
    reference algorithm, test infrastructure) on the same grid as the GPU arm,
    generated by the oracle's own generator (bitwise the GPU arm's grid,
    tests/test_oracle.py).  Edge list, incidence and boundary lists are built
    outside the timed regions, like the GPU plan.

    rows: or_metrics_mt (dual-free navs + edge volumes, all host threads, the
    serial loops' summation order -> same bits) over `steps` steps after
    `warmup`; serial dual-free step (or_navs_dualfree + or_volumes_edge, one
    thread) warm-up + `serial_reps`; serial traditional navs
    (or_navs_traditional) warm-up + `trad_reps` (0 skips it)."""
    from oracle.oracle import Oracle
    if config != "C5":
        raise ValueError("the CPU legs time the C5 family (oracle generator)")
    threads = threads or host_threads()
    O = Oracle()
    n = 256 // scale
    t0 = time.perf_counter()
    m = O.gen_tet_cube(n, amp=0.15, seed=42)
    t1 = time.perf_counter()
    e, o = O.build_edges(m)
    t2 = time.perf_counter()
    plan = O.plan(m, e, o)
    t3 = time.perf_counter()
    out = (np.empty(3 * e.shape[0]), np.empty(e.shape[0]), np.empty(m.num_nodes()))
    rows = {"grid": f"{n}^3 Kuhn cube, +-0.15h (seed 42), {m.num_elements()} tets, "
                    f"{e.shape[0]} edges", "n_elements": m.num_elements(),
            "n_nodes": m.num_nodes(), "n_edges": int(e.shape[0]),
            "n_boundary": m.num_boundary(),
            "host_cpu": cpu_model(), "host_threads": threads,
            "setup_s": {"gen": t1 - t0, "build_edges": t2 - t1, "plan": t3 - t2}}
    try:
        for _ in range(warmup):
            O.metrics_mt(plan, m.coords, threads, out)
        t0 = time.perf_counter()
        for _ in range(steps):
            O.metrics_mt(plan, m.coords, threads, out)
        dt = (time.perf_counter() - t0) / steps
    finally:
        O.plan_free(plan)
    rows["mt_step_ms"] = dt * 1e3
    rows["mt_tets_per_s"] = m.num_elements() / dt
    if serial_reps > 0 or trad_reps > 0:
        t0 = time.perf_counter()
        e2l, _, _ = O.edge_maps(m, e, o)
        rows["setup_s"]["edge_maps"] = time.perf_counter() - t0

        def best(fn, reps):
            fn()  # warm-up
            ts = []
            for _ in range(reps):
                a = time.perf_counter()
                fn()
                ts.append(time.perf_counter() - a)
            return min(ts) * 1e3, float(np.mean(ts)) * 1e3

        if serial_reps > 0:
            nv = O.navs_dualfree(m, e, o, e2l)
            rows["serial_dualfree_navs_ms"], _ = best(lambda: O.navs_dualfree(m, e, o, e2l),
                                                     serial_reps)
            rows["serial_edge_volumes_ms"], _ = best(lambda: O.volumes_edge(m, e, nv), serial_reps)
            st = rows["serial_dualfree_navs_ms"] + rows["serial_edge_volumes_ms"]
            rows["serial_step_ms"] = st
            rows["serial_tets_per_s"] = m.num_elements() / (st / 1e3)
            rows["serial_reps"] = serial_reps
        if trad_reps > 0:
            rows["serial_traditional_navs_ms"], _ = best(
                lambda: O.navs_traditional(m, e, o, e2l), trad_reps)
            rows["trad_reps"] = trad_reps
            if "serial_dualfree_navs_ms" in rows:
                rows["cpu_traditional_over_dualfree_navs"] = (
                    rows["serial_traditional_navs_ms"] / rows["serial_dualfree_navs_ms"])
                rows["paper_traditional_over_dualfree_navs"] = 2.16
    return rows


def run_reference(args, world, rank, dist):
    if rank != 0:
        return
    steps, warmup = args.steps, args.warmup
    rows = cpu_rows(args.config, args.scale, steps, warmup, args.serial_reps, args.trad_reps)
    value, th = rows["mt_tets_per_s"], rows["host_threads"]
    sample = (f"oracle/oracle.c or_metrics_mt (CPU restatement of the reference algorithm, "
              f"-O2 -ffp-contract=off, {th} threads, {rows['host_cpu']}) on the full "
              f"{args.config} grid ({rows['grid']}), dual-free navs + edge volumes, "
              f"{steps} steps after {warmup} warm-up; serial rows in cpu_rows")
    line = {"metric": METRIC, "value": value, "unit": "tets/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": steps, "warmup": warmup,
            "ms_per_step": rows["mt_step_ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, args.scale),
                       "n_elements": rows["n_elements"], "n_nodes": rows["n_nodes"],
                       "n_edges": rows["n_edges"], "n_boundary": rows["n_boundary"],
                       "nav_variant": "dual-free element loop, serial summation order",
                       "parallelism": f"host CPU, {th} threads",
                       "l2": "inputs larger than the host caches (no flush)"},
            "cpu_baseline": {"value": value, "unit": "tets/s", "cores": th, "kind": "port",
                             "sample": sample},
            "cpu_rows": rows,
            "e2e": {"value": value, "unit": "tets/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_name(config, scale):
    if config == "C5" and scale == 1:
        return "C5: 256^3 Kuhn cube, +-0.15h jitter (seed 42)"
    return f"{config}/scale {scale}"


# ---------------------------------------------------------------- GPU arm
def run_ours(args, world, rank, local, dist):
    import torch
    from paper_2502_00778_b200 import Engine, _lib, meshgen

    torch.cuda.set_device(local)
    t0 = time.perf_counter()
    mesh = meshgen.baseline_config(args.config, args.scale)
    gen_s = time.perf_counter() - t0
    eng = Engine(local)
    eng.set_mesh(mesh)
    # K1 edge extraction (outside the SPEC timed region; reported separately)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stream = torch.cuda.ExternalStream(eng.stream())
    ev0.record(stream)
    ne = eng.build_edges()
    ev1.record(stream)
    torch.cuda.synchronize()
    edges_ms_first = ev0.elapsed_time(ev1)  # includes the buffers' cudaMalloc
    ev0.record(stream)
    ne = eng.build_edges()  # steady state (re-extraction, buffers resident)
    ev1.record(stream)
    torch.cuda.synchronize()
    edges_ms = ev0.elapsed_time(ev1)
    variant = _lib.DM_VARIANT_SCATTER if args.variant == "scatter" else _lib.DM_VARIANT_GATHER
    DF, TR, EDGE = _lib.DM_NAV_DUALFREE, _lib.DM_NAV_TRADITIONAL, _lib.DM_VOL_EDGE
    # derived structures (boundary lists, incoming CSR, the ring plan) are
    # built by the first call: that one-time cost is reported as plan_ms
    torch.cuda.synchronize()
    t_plan = time.perf_counter()
    eng.navs(DF, variant)
    eng.volumes(EDGE)
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - t_plan) * 1e3
    # the same plan rebuilt on a warm context (edge re-extraction drops it;
    # buffers stay allocated): the cost without first-touch cudaMalloc stalls
    eng.build_edges()
    torch.cuda.synchronize()
    t_plan = time.perf_counter()
    eng.navs(DF, variant)
    eng.volumes(EDGE)
    torch.cuda.synchronize()
    replan_ms = (time.perf_counter() - t_plan) * 1e3
    bmask = eng.boundary_node_mask()
    bd = mesh.boundary.reshape(-1, mesh.dim)
    if mesh.dim == 3:
        pairs = np.concatenate([bd[:, [0, 1]], bd[:, [1, 2]], bd[:, [2, 0]]])
    else:
        pairs = bd[:, [0, 1]]
    pairs = np.sort(pairs, axis=1).astype(np.int64)
    n_bnd_edges = int(np.unique(pairs[:, 0] * (1 << 32) + pairs[:, 1]).size)
    B = algorithmic_bytes(mesh, ne, int(bmask.sum()), n_bnd_edges)
    peak, peak_kind = hbm_peak()

    def step(evs=None):
        if evs is not None:
            evs[0].record(stream)
        eng.navs(DF, variant)
        if evs is not None:
            evs[1].record(stream)
        eng.volumes(EDGE)
        if evs is not None:
            evs[2].record(stream)

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(args.warmup):
        step()
    # keep warming up until nvidia-smi is producing samples, so the timed
    # region is covered by clock samples (bounded wait)
    t_wait = time.perf_counter()
    while not clocks.live() and time.perf_counter() - t_wait < 5.0:
        for _ in range(10):
            step()
        torch.cuda.synchronize()
    torch.cuda.synchronize()
    K = args.steps
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    launches0 = eng.launches()
    # the library records CUDA events around each kernel phase of the K timed
    # steps on its own stream (no synchronisation inside the region): the
    # per-kernel times below come from the timed region itself
    eng.set_step_timing(K)
    barrier(dist)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host_t0 = time.time()
    start.record(stream)
    for k in range(K):
        step(evs[k])
    end.record(stream)
    torch.cuda.synchronize()
    host_t1 = time.time()
    barrier(dist)
    clk = clocks.stop(host_t0, host_t1)
    launches = eng.launches() - launches0
    total_ms = start.elapsed_time(end)
    total_ms = max_over_ranks(dist, total_ms, device=torch.device("cuda", local))
    ms_step = total_ms / K
    nav_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    vol_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    value = world * K * mesh.num_elements() / (total_ms / 1e3)

    # the dominant kernel alone: the library's own CUDA events on its stream
    # around the element-loop launch (slot 0), the boundary pass (1) and the
    # volume kernel (2), recorded during the K timed steps
    kt = eng.step_timings(K)
    eng.set_timing(False)
    assert kt.shape[0] == K, kt.shape
    elem_ms, bnd_ms, kvol_ms = (float(np.mean(kt[:, i])) for i in range(3))
    # the same phases with a synchronisation after every step (the GPU idles
    # between steps: cooler, often faster clocks), for comparison only
    eng.set_timing(True)
    ks = []
    for _ in range(min(K, 10)):
        step()
        ks.append(eng.timings())
    eng.set_timing(False)
    ks = np.array(ks)

    # GPU traditional comparator (north_star (e)), same harness, not the headline
    for _ in range(max(1, args.warmup // 2)):
        eng.navs(TR, _lib.DM_VARIANT_GATHER)
    torch.cuda.synchronize()
    t_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(K)]
    for k in range(K):
        t_ev[k][0].record(stream)
        eng.navs(TR, _lib.DM_VARIANT_GATHER)
        t_ev[k][1].record(stream)
        eng.volumes(EDGE)
        t_ev[k][2].record(stream)
    torch.cuda.synchronize()
    trad_ms = float(np.mean([e[0].elapsed_time(e[2]) for e in t_ev]))
    trad_navs_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in t_ev]))

    # e2e: the public C-ABI step with host buffers (pinned), H2D coords + D2H navs/volumes
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        nb_c = mesh.coords.nbytes
        nb_n = 8 * mesh.dim * ne
        nb_v = 8 * mesh.num_nodes()
        hp = [C.c_void_p() for _ in range(3)]
        for p, nb in zip(hp, (nb_c, nb_n, nb_v)):
            if _lib.capi().dm_host_alloc(nb, C.byref(p)) != 0:
                raise MemoryError("pinned allocation failed")
        hc = np.ctypeslib.as_array(C.cast(hp[0], C.POINTER(C.c_double)), shape=(mesh.coords.size,))
        hc[:] = mesh.coords
        dp = lambda p: C.cast(p, C.POINTER(C.c_double))  # noqa: E731
        for _ in range(2):
            eng.metrics_host(dp(hp[0]), DF, variant, EDGE, dp(hp[1]), dp(hp[2]))
        # one synchronous step (copy-in, kernels, copy-out back to back)
        barrier(dist)
        t0 = time.perf_counter()
        eng.metrics_host(dp(hp[0]), DF, variant, EDGE, dp(hp[1]), dp(hp[2]))
        t_sync = time.perf_counter() - t0
        # the pipelined loop: every step still copies its coordinates in and
        # its navs + volumes out; step i+1's copy-in and kernels overlap step
        # i's copy-out (full-duplex PCIe, two device output buffers)
        barrier(dist)
        t0 = time.perf_counter()
        ke = max(3, K // 2)
        for _ in range(ke):
            eng.metrics_host_async(dp(hp[0]), DF, variant, EDGE, dp(hp[1]), dp(hp[2]))
        eng.sync()
        t_e2e = (time.perf_counter() - t0) / ke
        t_e2e = max_over_ranks(dist, t_e2e, device=torch.device("cuda", local))
        t_sync = max_over_ranks(dist, t_sync, device=torch.device("cuda", local))
        e2e = {"value": world * mesh.num_elements() / t_e2e, "unit": "tets/s",
               "h2d_bytes_per_step": nb_c, "d2h_bytes_per_step": nb_n + nb_v,
               "ms_per_step": t_e2e * 1e3, "steps": ke,
               "ms_single_synchronous_step": t_sync * 1e3,
               "api": "dm_metrics_host_async x steps + dm_sync (include/dm_capi.h), pinned "
                      "host buffers; wall clock from the first call to the final sync"}
        for p in hp:
            _lib.capi().dm_host_free(p)

    kernel_bytes = B["elem"]
    achieved = kernel_bytes / (elem_ms / 1e3) / 1e9
    step_achieved = B["metrics"] / (ms_step / 1e3) / 1e9
    # each kernel against the bytes its own design moves,
    # beside the canonical SURVEY 8(d) bytes above
    D, nv = mesh.dim, mesh.num_nodes()
    pb = eng.plan_bytes()
    design = {}
    if pb["tiles"]:
        d_elem = (pb["codes"] + pb["meta_runs"] + 8 * D * nv + 8 * D * ne + 8 * ne)
        design["element_loop"] = {
            "bytes": d_elem, "ms": elem_ms, "frac": d_elem / (elem_ms / 1e3) / 1e9 / peak,
            "parts": {"ring_codes": pb["codes"], "tile_meta_runs": pb["meta_runs"],
                      "coords_once": 8 * D * nv, "navs_rows": 8 * D * ne, "s_terms": 8 * ne},
            "table_fill_from_l2_or_hbm": pb["table_fill"],
            "note": "row tiles: codes + run descriptors + coordinates once + navs + s"}
    d_vol = 4 * (nv + 1) + 4 * ne + 4 * (nv + 1) + 8 * ne + 8 * nv
    design["volumes"] = {"bytes": d_vol, "ms": kvol_ms,
                         "frac": d_vol / (kvol_ms / 1e3) / 1e9 / peak,
                         "note": "in_ptr + in_list + origin CSR + s once + V"}
    traffic = None
    prof = os.path.join(ROOT, "profiles", "latest_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("navs_kernel_dram_bytes")
        except Exception:
            traffic = None

    cpu = None
    crow = None
    if rank == 0 and world == 1 and not args.no_cpu and args.config == "C5":
        crow = cpu_rows(args.config, args.scale, args.cpu_steps, 1, args.serial_reps,
                        args.trad_reps)
        cpu = {"value": crow["mt_tets_per_s"], "unit": "tets/s", "cores": crow["host_threads"],
               "kind": "port",
               "sample": f"oracle/oracle.c or_metrics_mt ({crow['host_threads']} threads, "
                         f"{crow['host_cpu']}) on the same full grid ({crow['grid']}), "
                         f"dual-free navs + edge volumes, {args.cpu_steps} steps after 1 "
                         f"warm-up, {crow['mt_step_ms']:.1f} ms/step; serial rows in "
                         f"cpu_rows"}
        if "serial_step_ms" in crow:
            cpu["serial_1_thread"] = {"value": crow["serial_tets_per_s"], "unit": "tets/s",
                                      "cores": 1, "ms_per_step": crow["serial_step_ms"]}
            crow["gpu_step_over_serial_step"] = crow["serial_step_ms"] / ms_step
        crow["gpu_step_over_mt_step"] = crow["mt_step_ms"] / ms_step
        if "serial_traditional_navs_ms" in crow:
            crow["gpu_traditional_over_dualfree_navs"] = trad_navs_ms / nav_ms

    cpp_api = None
    if rank == 0 and world == 1 and not args.no_cpp_api and args.config == "C5":
        # the reference-facing C++ API (dualmesh::compute_metrics etc.) with
        # std::vector buffers, timed by its own tool on a fresh process
        exe = os.path.join(ROOT, "tools", "_build", "cpp_api_bench")
        if os.path.exists(exe):
            try:
                r = subprocess.run([exe, str(256 // args.scale)], capture_output=True, text=True,
                                   timeout=600)
                cpp_api = json.loads(r.stdout.strip().splitlines()[-1])
            except Exception as ex:  # reported, not fatal
                cpp_api = {"error": repr(ex)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tets/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(args.config, args.scale),
                       "n_elements": mesh.num_elements(), "n_nodes": mesh.num_nodes(),
                       "n_edges": ne, "n_boundary": mesh.num_boundary(),
                       "nav_variant": args.variant,
                       "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                       "l2": "inputs larger than L2 (no flush): "
                             f"{B['metrics'] / 1e9:.2f} GB algorithmic per step"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("k_navs_row (K2 dual-free element loop on row tiles, "
                                    "scale pass and s_e fused)" if pb["tiles"] else
                                    "k_navs_ring_pipe (K2 dual-free element loop on Morton "
                                    "tiles, scale pass and s_e fused)"),
                         "bytes_per_launch": kernel_bytes, "ms_per_launch": elem_ms,
                         "peak_source": peak_kind},
            "design_roofline": design,
            "step_roofline": {"achieved": step_achieved, "frac": step_achieved / peak,
                              "bytes_per_step": B["metrics"], "unit": "GB/s",
                              "nav_ms": nav_ms, "vol_ms": vol_ms,
                              "kernels_ms": {"element_loop": elem_ms, "boundary": bnd_ms,
                                             "volumes": kvol_ms,
                                             "source": "CUDA events on the library stream "
                                                       "inside the timed region, mean of the "
                                                       "K steps"},
                              "kernels_ms_synchronised_steps": {
                                  "element_loop": float(np.mean(ks[:, 0])),
                                  "boundary": float(np.mean(ks[:, 1])),
                                  "volumes": float(np.mean(ks[:, 2]))}},
            "cpu_baseline": cpu,
            "cpu_rows": crow,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "extra": {"roofline_vs_nominal": {
                          "nominal_gbs": 8000.0, "element_loop_frac": achieved / 8000.0,
                          "step_frac": B["metrics"] / (ms_step / 1e3) / 1e9 / 8000.0},
                      "throughput": {
                          "step_tets_per_s": value, "step_edges_per_s": world * K * ne / (total_ms / 1e3),
                          "element_loop_edges_per_s": ne / (elem_ms / 1e3),
                          "edge_extraction_tets_per_s": mesh.num_elements() / (edges_ms / 1e3),
                          "edge_extraction_edges_per_s": ne / (edges_ms / 1e3)},
                      "edges_ms": edges_ms, "edges_ms_first_call": edges_ms_first,
                      "plan_ms_first_call": plan_ms, "plan_ms_rebuild": replan_ms,
                      "plan": eng.plan_info(), "edges_bytes": B["edges"],
                      "edges_GBps": B["edges"] / (edges_ms / 1e3) / 1e9,
                      "full_pipeline_device_ms": edges_ms + replan_ms,
                      "full_pipeline_note": "K1 edge extraction (warm) + plan rebuild + one "
                                            "step, topology fresh, data resident",
                      "plan_steps_to_amortise": (replan_ms - ms_step) / ms_step,
                      "cpp_api": cpp_api,
                      "traditional_ms_per_step": trad_ms,
                      "traditional_navs_ms": trad_navs_ms, "dualfree_navs_ms": nav_ms,
                      "gpu_speedup_dualfree_over_traditional": trad_ms / ms_step,
                      "gpu_traditional_over_dualfree_navs": trad_navs_ms / nav_ms,
                      "meshgen_s": gen_s},
        }
        print(json.dumps(line), flush=True)
    eng.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--variant", choices=["gather", "scatter"], default="gather")
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--serial-reps", type=int, default=3,
                    help="serial CPU dual-free step: warm-up + this many reps (0 skips)")
    ap.add_argument("--trad-reps", type=int, default=1,
                    help="serial CPU traditional navs: warm-up + this many reps (0 skips)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpp-api", action="store_true")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference(args, world, rank, dist)
        else:
            run_ours(args, world, rank, local, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
