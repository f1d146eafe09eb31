#!/usr/bin/env python
"""Benchmark: time-to-maximum-matching on B200 (BASELINE.json metric).

Default workload (N=1): C5 = the largest synthetic graph of BASELINE.json
(configs[4]; north_star puts the 1-GPU targets on it): the reference's own
generate_random_bipartite(1e8, 1e8, 16.0, seed 5), 1.6e9 edges, APFB-GPUBFS-WR
from the reference's first-fit initial matching (the reference methodology:
cheap_matching outside the timed region, bench.cpp:52-63). One *step* = one
complete run to the maximum matching from the same initial matching, inputs
resident in HBM.

  value     = graph edges / time-to-maximum-matching   (edges/s, higher is better)
  e2e       = same metric through the public C-ABI call with pinned host
              buffers: graph upload + init H2D + matching + result D2H per step
  roofline  = algorithmic bytes of the driver kernel / its CUDA-event time,
              against the measured HBM copy bandwidth (MEASURED_PEAKS.json)
  cpu_baseline / --impl reference = the reference's own CPU implementation
              (oracle/_ref: /root/reference sources compiled unmodified),
              apfb-wr-ct under Schedule::parallel(all host cores)

The reference arm builds its input with oracle/gen_oracle.cpp (a restatement
of the same generators) and never loads the product library. Each of its steps
is one full run of the same workload; at C5 one run takes about a minute on 16
cores, so it times as many steps as fit its --ref-budget-s (reported as
`steps`, with `steps_requested`).

Multi-GPU (torchrun, N>1): by default the workload is 1-D partitioned by
column across the ranks (strong scaling, paper_1303_1379_b200/partition.py):
the multi-GPU engine runs the whole driver as one persistent launch per rank,
claims resolved at the row's owner and winner columns stored into their
owner's inbox over peer memory (CUDA IPC / NVLink), the level barrier
spanning the team. --mode replicas instead solves one independent replica per
rank (weak scaling, no collective). Timing is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL's "NCCL version ..." banner goes to stdout; the contract is one JSON line there
if os.environ.get("NCCL_DEBUG", "VERSION").upper() == "VERSION":
    os.environ["NCCL_DEBUG"] = "WARN"

METRIC = "time-to-maximum-matching (ms) and traversed edges/sec; % of HBM roofline"

# name -> (description, builder kwargs)
CONFIGS = {
    "C1": "uniform random 100K x 100K, avg degree 8, seed 1 (reference generator)",
    "C2": "planted perfect matching 10M x 10M, avg degree 16, seed 2024",
    "C3": "bipartite R-MAT scale 24, edge factor 16, (0.57,0.19,0.19), permuted, seed 2024",
    "C4": "banded (band 3) 20M x 20M, 5% rows deleted, permuted, seed 12345",
    "C5": "uniform random 100M x 100M, avg degree 16, seed 5 (reference generator)",
}

ALGOS = {  # id -> (shortest, kernel, improved)  algorithms.cpp:19-27
    "apfb-wr": (False, 1, False),
    "apfb-gpubfs": (False, 0, False),
    "apsb-wr": (True, 1, True),
    "apsb-gpubfs": (True, 0, False),
}


GRAPH_FILE = None  # --graph: a user matrix instead of a synthetic config


def build_graph(name: str, scale_div: int = 1):
    import paper_1303_1379_b200 as bm
    if name == "file":  # maximum unknown up front: the GPU certificate and the reference arm check it
        path = GRAPH_FILE
        return (bm.load_csc(path) if path.endswith(".bcsc") else bm.load_matrix_market(path)), None
    if name == "C1":
        return bm.generate_random_bipartite(100_000, 100_000, 8.0, 1), 99_961
    if name == "C2":
        n = 10_000_000 // scale_div
        return bm.generate_planted(n, 16.0, 2024), n
    if name == "C3":
        return bm.generate_rmat(24, 16.0, 2024), None
    if name == "C4":
        g, live = bm.generate_banded(20_000_000 // scale_div, 3, 0.05, 12345)
        return g, live
    if name == "C5":
        n = 100_000_000 // scale_div
        return bm.generate_random_bipartite(n, n, 16.0, 5), (99_999_986 if scale_div == 1 else None)
    raise SystemExit(f"unknown config {name}")


def build_graph_oracle(name: str, scale_div: int = 1):
    """The same graphs as build_graph, built by oracle/gen_oracle.cpp (the
    reference arm must not map the product library)."""
    from oracle import Generators, Reference, OGraph
    gen = Generators()
    if name == "file":  # the reference's own reader (matrix_market.cpp) through oracle/_ref
        if GRAPH_FILE.endswith(".bcsc"):
            raise SystemExit("--impl reference reads Matrix Market files only")
        with open(GRAPH_FILE, "rb") as f:
            st = Reference().read_matrix_market(f.read())
        if st[0] != "ok":
            raise SystemExit(f"reference reader failed: {st}")
        return OGraph(st[1], st[2], st[3], st[4], os.path.basename(GRAPH_FILE)), None
    if name == "C1":
        return gen.uniform(100_000, 100_000, 8.0, 1), 99_961
    if name == "C2":
        n = 10_000_000 // scale_div
        return gen.planted(n, 16.0, 2024), n
    if name == "C3":
        return gen.rmat(24, 16.0, 2024), None
    if name == "C4":
        return gen.banded(20_000_000 // scale_div, 3, 0.05, 12345)
    if name == "C5":
        n = 100_000_000 // scale_div
        return gen.uniform(n, n, 16.0, 5), (99_999_986 if scale_div == 1 else None)
    raise SystemExit(f"unknown config {name}")


def workload_config(args, g) -> dict:
    """The `config` object, identical in both arms (impl-specific keys live outside it)."""
    return {"workload": f"{args.config}: {CONFIGS[args.config]}" +
                        (f" (1/{args.scale_div} scale)" if args.scale_div != 1 else ""),
            "nc": g.nc, "nr": g.nr, "edges": g.num_edges(),
            "init": "first-fit cheap_matching (matching.cpp:13-26), computed before timing",
            "l2": f"GPU arm flushes L2 between steps ({args.flush_mb} MiB write)"}


def data_kind() -> str:
    return f"file {os.path.basename(GRAPH_FILE)}" if GRAPH_FILE else "synthetic"


def known_answers():
    p = os.path.join(ROOT, "tests", "golden", "known_answers.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def random_access_ceiling(trav, k_ms):
    """The path's other ceiling: every traversed edge needs at least one random
    4-byte access to the row state, which on B200 runs at the rate the
    microbenchmark (scripts/ubench_gather.cu, committed as
    profiles/ubench_gather.jsonl) measures for the C5-sized table, not at the
    HBM copy bandwidth. t_min = traversed edges / best gather rate."""
    path = os.path.join(ROOT, "profiles", "ubench_gather.jsonl")
    if not os.path.exists(path):
        return None
    rows = [json.loads(l) for l in open(path) if l.strip()]
    big = max(r["table_mb"] for r in rows)
    best = {}
    for r in rows:
        if r["table_mb"] == big:
            best[r["kind"]] = max(best.get(r["kind"], 0.0), r["gps"])
    g = best.get("gather")
    if not g:
        return None
    t_min = trav / (g * 1e9) * 1e3
    return {"table_mb": big, "gather_gps": g, "claim_gps": best.get("claim"), "atomic_gps": best.get("atomicOr"),
            "traversed_edges": trav, "t_min_ms": t_min, "frac": t_min / k_ms,
            "model": "one random 4-byte row-state gather per traversed edge at the best measured gather rate",
            "source": "profiles/ubench_gather.jsonl (scripts/ubench_gather.cu on this pool's B200)"}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML during the timed region."""

    REASONS = [
        ("gpu_idle", "nvmlClocksEventReasonGpuIdle"),
        ("applications_clocks_setting", "nvmlClocksEventReasonApplicationsClocksSetting"),
        ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
        ("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
        ("sync_boost", "nvmlClocksEventReasonSyncBoost"),
        ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
        ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
        ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"),
    ]

    def __init__(self, device: int, period_s: float = 0.01):
        self.period = period_s
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _loop(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, attr in self.REASONS:
                    bit = getattr(nv, attr, 0)
                    if bit and (mask & bit) and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


_JSON_FD = None  # set while library banners (NCCL) are diverted away from stdout


def emit(obj):
    line = json.dumps(obj) + "\n"
    if _JSON_FD is not None:
        os.write(_JSON_FD, line.encode())
    else:
        print(line, end="", flush=True)


def divert_stdout():
    """Route fd 1 to stderr for the rest of the run (NCCL prints its version banner
    on stdout when its communicator is created); emit() keeps the real stdout."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


_REF_CACHE = {}


def cpu_reference_run(g, init, threads_label="parallel"):
    """The reference's apfb-wr-ct (make_algorithm + Schedule::parallel, kernel_grid.cpp:127-131)."""
    from oracle import Reference, have_reference
    if have_reference():
        ref = _REF_CACHE.setdefault("ref", Reference())
        key = id(g)
        if _REF_CACHE.get("key") != key:
            _REF_CACHE["graph"] = ref.from_csc(g)  # BipartiteCsr copy, not timed
            _REF_CACHE["key"] = key
        rg = _REF_CACHE["graph"]
        r, c, ct, secs = rg.run("apfb-wr-ct", init.rmatch, init.cmatch, threads_label)
        return {"kind": "reference", "cores": ref.hw_threads(), "seconds": secs,
                "cardinality": int((r >= 0).sum()), "counters": ct}
    from oracle import Oracle
    orc = Oracle()
    t0 = time.perf_counter()
    st, r, c, ct = orc.driver(g, init.rmatch, init.cmatch, tot=65536, kernel=1)
    secs = time.perf_counter() - t0
    return {"kind": "port", "cores": 1, "seconds": secs, "cardinality": int((r >= 0).sum()), "counters": ct}


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    apfb-wr-ct under Schedule::parallel(all host threads), kernel_grid.cpp:127-131,
    timed as bench.cpp:52-63) on the same workload. Nothing from the product
    package is imported or loaded here."""
    world, rank, local = dist_env()
    if rank != 0:
        return 0
    from oracle import Generators, have_reference
    t_gen = time.perf_counter()
    g, known = build_graph_oracle(args.config, args.scale_div)
    if known is None:
        known = known_answers().get(f"{args.config}/div{args.scale_div}")
    r0, c0 = Generators().first_fit(g)

    class _Init:
        rmatch, cmatch = r0, c0
    t_gen = time.perf_counter() - t_gen
    E = g.num_edges()
    budget = args.ref_budget_s
    wall0 = time.perf_counter()
    probe = cpu_reference_run(g, _Init)  # first run: warm-up, and the per-step cost estimate
    t1 = probe["seconds"]
    cards = [probe["cardinality"]]
    warm = min(args.warmup, 1)
    if t1 * (args.warmup - 1 + args.steps) <= budget:
        for _ in range(max(0, args.warmup - 1)):
            cards.append(cpu_reference_run(g, _Init)["cardinality"])
        warm = max(args.warmup, 1)
        steps = args.steps
    else:  # one step is a full run; time as many as fit the budget
        steps = max(1, min(args.steps, int(budget // max(t1, 1e-9))))
    times = []
    for _ in range(steps):
        res = cpu_reference_run(g, _Init)
        times.append(res["seconds"])
        cards.append(res["cardinality"])
    kind, cores = res["kind"], res["cores"]
    t = statistics.mean(times)
    value = E / t
    sample = (f"{steps} full {args.config} run(s) ({g.nc}x{g.nr}, {E} edges) of apfb-wr-ct parallel:{cores} "
              f"from first-fit; {warm} untimed warm-up run(s)")
    emit({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
        "steps": steps, "steps_requested": args.steps, "warmup": warm, "warmup_requested": args.warmup,
        "ms_per_step": t * 1e3, "ms_per_step_min": min(times) * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": data_kind(),
        "config": workload_config(args, g),
        "algorithm": "apfb-wr-ct (reference CPU, oracle/_ref)" if have_reference() else "apfb-wr (C port, serial)",
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": cores, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "time_to_max_matching_ms": t * 1e3, "cardinality": cards[-1],
        "parity": {"known_answer": known, "ok": (known is None or all(c == known for c in cards))},
        "generation_s": t_gen, "wall_s": time.perf_counter() - wall0,
    })
    return 0


def run_partitioned(args):
    """N ranks, one GPU each (torchrun), one column slice each:
    the multi-GPU engine (csrc/bm_mg.cu) runs the whole driver as one launch
    per rank over peer memory. value = graph edges / time (max over ranks)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1303_1379_b200 as bm
    from paper_1303_1379_b200.partition import DistTransport, GpuRank, PartitionedMatcher

    world, rank, local = dist_env()
    divert_stdout()
    ndev = max(1, torch.cuda.device_count())
    local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("gloo", rank=rank, world_size=world)  # setup messages only (no data path)
    t_gen = time.perf_counter()
    g, known = build_graph(args.config, args.scale_div)
    if known is None:
        known = known_answers().get(f"{args.config}/div{args.scale_div}")
    init = bm.cheap_matching(g)
    t_gen = time.perf_counter() - t_gen
    E = g.num_edges()
    shortest, kernel, improved = ALGOS[args.algo]
    kernel = bm.BfsKernel(kernel)
    # ranks sharing a device (more ranks than GPUs) cannot co-run their persistent kernels across processes
    if world > ndev:
        raise SystemExit(f"{world} ranks on {ndev} GPU(s): the multi-GPU engine needs one GPU per rank")
    x = DistTransport()
    rk = GpuRank(local, rank, world)
    stream = torch.cuda.current_stream(dev)
    rk.set_stream(stream.cuda_stream)
    pm = PartitionedMatcher(rk, x)
    pulled = args.bottom_up != "off"
    t_up = time.perf_counter()
    pm.upload(g, row_index=pulled)
    t_up = time.perf_counter() - t_up
    bu = {"auto": "auto", "on": "on", "off": "off"}[args.bottom_up]

    def step():
        return pm.match(init, shortest=shortest, kernel=kernel, improved=improved, bottom_up=bu)

    res = step()
    m = pm.gather()
    parity_ok = known is None or res.cardinality == known
    for _ in range(args.warmup):
        step()
    x.barrier()
    kms, cards, ph = [], [], []
    sampler = ClockSampler(local)
    with sampler:
        for _ in range(args.steps):
            r = step()  # load + barrier + launch + finish; the kernel time is the run
            kms.append(r.kernel_ms)
            cards.append(r.cardinality)
            ph.append(r.phases)
            parity_ok = parity_ok and (known is None or r.cardinality == known)
    t_ms = x.allreduce_max(statistics.mean(kms))
    trav = x.allreduce_sum(sum(c.edges_traversed for c in r.counters))
    cexp = x.allreduce_sum(sum(c.columns_scanned for c in r.counters))
    nvis = x.allreduce_sum(sum(c.columns_visited for c in r.counters))
    steps_walk = x.allreduce_sum(sum(c.walk_steps for c in r.counters))

    # end to end through the public API: each rank uploads its slice from pinned host memory,
    # matches, and reads its rows and columns back
    e2e = None
    if not args.no_e2e:
        lo, hi = pm.cb[rank], pm.cb[rank + 1]
        rlo, rhi = pm.rb[rank], pm.rb[rank + 1]
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        cx = pin(g.cxadj[lo:hi + 1] - g.cxadj[lo])
        adj = pin(g.cadj[int(g.cxadj[lo]):int(g.cxadj[hi])])
        # pinned host buffers for this rank's initial-matching slices and results, as the
        # single-GPU e2e uses
        r_sl, c_sl = pin(init.rmatch[rlo:rhi]), pin(init.cmatch[lo:hi])
        out_r, out_c = pin(np.empty(rhi - rlo, np.int32)), pin(np.empty(hi - lo, np.int32))
        e_ms = []
        for i in range(args.warmup + args.steps):
            x.barrier()
            t0 = time.perf_counter()
            pm.upload(g, row_index=pulled, slices=(cx.numpy(), adj.numpy()))
            pm.match(init, shortest=shortest, kernel=kernel, improved=improved, bottom_up=bu,
                     slices=(r_sl.numpy(), c_sl.numpy()))
            rs, cs = rk.download(out=(out_r.numpy(), out_c.numpy()))
            t1 = time.perf_counter()
            if i >= args.warmup:
                e_ms.append(1e3 * (t1 - t0))
        e_max = x.allreduce_max(statistics.mean(e_ms))
        h2d = x.allreduce_sum(int(cx.numel()) * 8 + int(adj.numel()) * 4 + 4 * ((pm.rb[rank + 1] - pm.rb[rank]) +
                                                                             (hi - lo)))
        d2h = 4 * (g.nr + g.nc)
        e2e = {"value": E / (e_max / 1e3), "unit": "edges/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": e_max, "note": "wall clock per rank (max over ranks): slice upload from host, "
                                             "row index, initial matching, the run, result download"}
    if rank == 0:
        eng = bm.Engine(local)  # GPU Berge certificate of the gathered result
        eng.upload(g)
        viol, ismax, vcard = eng.verify(g, m)
        g_ok = bool(viol == 0 and ismax and vcard == res.cardinality)
        del eng
        parity_ok = parity_ok and g_ok
        cpu = None
        if not args.no_cpu_baseline:
            cr = cpu_reference_run(g, init)
            cpu = {"value": E / cr["seconds"], "unit": "edges/s", "cores": cr["cores"], "kind": cr["kind"],
                   "sample": f"one full {args.config} run ({E} edges) of apfb-wr-ct on the host",
                   "seconds": cr["seconds"], "cardinality": cr["cardinality"]}
            parity_ok = parity_ok and cr["cardinality"] == res.cardinality
        wr = 1 if kernel == bm.BfsKernel.GpubfsWr else 0
        b_units = 12 * trav + (20 + 8 * wr) * cexp + (8 + 4 * wr) * nvis + 20 * steps_walk
        peak, peak_src = measured_peak()
        achieved = b_units / (t_ms / 1e3) / 1e9
        emit({
            "metric": METRIC, "value": E / (t_ms / 1e3), "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": data_kind(),
            "config": workload_config(args, g),
            "algorithm": f"{args.algo}-b200-multigpu",
            "parallelism": f"1-D column partition x{world}: one persistent launch per rank, claims at the row's "
                           "owner and winners into the column's owner over peer memory (CUDA IPC / NVLink)",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                         "frac": achieved / (peak * world), "traffic": None, "peak_source": peak_src + f" x {world}",
                         "kernel": "bmg::driver_kernel (persistent, whole run, every rank)",
                         "algorithmic_bytes_per_launch": b_units},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": args.steps * world,
            "clocks": sampler.summary(),
            "time_to_max_matching_ms": t_ms, "cardinality": cards[-1] if cards else res.cardinality,
            "phases": ph, "bfs_levels": res.levels,
            "parity": {"known_answer": known, "gpu_verify": g_ok, "ok": bool(parity_ok)},
            "generation_s": t_gen, "upload_s": t_up,
        })
    x.barrier()
    dist.destroy_process_group()
    return 0


def run_b200(args):
    import numpy as np
    import torch
    import paper_1303_1379_b200 as bm

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        divert_stdout()
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        dist = None
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if dist is not None:
            dist.barrier()

    t_gen = time.perf_counter()
    g, known = build_graph(args.config, args.scale_div)
    kn = known_answers()
    if known is None:
        known = kn.get(f"{args.config}/div{args.scale_div}")
    init = bm.cheap_matching(g)
    t_gen = time.perf_counter() - t_gen
    E = g.num_edges()
    shortest, kernel, improved = ALGOS[args.algo]
    kernel = bm.BfsKernel(kernel)

    eng = bm.Engine(local)
    eng.set_stream(stream.cuda_stream)
    t_upload = time.perf_counter()
    eng.upload(g)
    t_upload = 1e3 * (time.perf_counter() - t_upload)
    eng.load_matching(init)
    flush = torch.empty(args.flush_mb << 20, dtype=torch.uint8, device=dev)

    # the traversal direction this run measures: auto resolves per graph at upload; a
    # qualifying graph gets its row index with the upload (graph preparation, like the
    # CSC upload itself outside `value`; timed and reported as row_index_ms)
    auto_level = eng.bottom_up_auto()
    pulled = args.bottom_up == "on" or (args.bottom_up == "auto" and auto_level > 0)
    row_index_ms = []

    def prepare():
        if pulled:
            t = time.perf_counter()
            eng.prepare_row_index()
            row_index_ms.append(1e3 * (time.perf_counter() - t))
    prepare()

    def one_step(bottom_up=pulled):
        return eng.run(shortest=shortest, kernel=kernel, improved=improved, bottom_up=bottom_up)

    # correctness of the measured configuration (GPU Berge certificate)
    card, ct, done = one_step()
    m = eng.download()
    viol, ismax, vcard = eng.verify(g, m)
    parity_ok = bool(done and viol == 0 and ismax and vcard == card and (known is None or card == known))
    eng.upload(g, force=True)
    eng.load_matching(init)
    prepare()

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    step_ms, kern_ms, launches, cards = [], [], 0, []
    counters = None
    step_counters = []  # per timed step: the roofline uses the mean work over the same steps as the mean time
    sampler = ClockSampler(local)
    wall0 = time.perf_counter()
    with sampler:
        for _ in range(args.steps):
            flush.fill_(1)  # > L2 (126 MB): every step starts cold
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            card, counters, done = one_step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            step_counters.append(counters)
            kms, nl = eng.last_kernel_time()
            kern_ms.append(kms)
            launches += nl
            cards.append(card)
            parity_ok = parity_ok and done and (known is None or card == known)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    wall = time.perf_counter() - wall0
    t_ms = statistics.mean(step_ms)
    k_ms = statistics.mean(kern_ms)
    if dist is not None:
        t = torch.tensor([t_ms, k_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms, k_ms = float(t[0]), float(t[1])

    # ---- the other traversal direction, measured the same way (reported, not the headline) ----
    alt = None
    if world == 1 and not args.no_alt:
        t_idx = time.perf_counter()
        one_step(not pulled)  # builds the row index on first use
        torch.cuda.synchronize(dev)
        t_idx = time.perf_counter() - t_idx
        a_ms, a_ph = [], []
        for _ in range(max(3, args.steps // 2)):
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            acard, act, adone = one_step(not pulled)
            e1.record(stream)
            e1.synchronize()
            a_ms.append(e0.elapsed_time(e1))
            a_ph.append(act.outer_iterations)
            parity_ok = parity_ok and adone and (known is None or acard == known)
        alt = {"bottom_up": not pulled, "ms_per_step": statistics.mean(a_ms),
               "phases": a_ph, "first_call_s": t_idx}

    # ---- end to end through the public API, pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
        cx_p, adj_p = pin(g.cxadj), pin(g.cadj)
        gp = bm.BipartiteCsr(g.nc, g.nr, cx_p.numpy(), adj_p.numpy(), g.name)
        r_p = torch.empty(g.nr, dtype=torch.int32).pin_memory()
        c_p = torch.empty(g.nc, dtype=torch.int32).pin_memory()
        ms_list = []
        eng2 = bm.Engine(local)
        eng2.set_stream(stream.cuda_stream)
        eng2.bottom_up = {"auto": "auto", "on": True, "off": False}[args.bottom_up]
        for i in range(args.warmup + args.steps):
            r_p.numpy()[:] = init.rmatch
            c_p.numpy()[:] = init.cmatch
            mstate = bm.MatchingState.__new__(bm.MatchingState)
            mstate.rmatch, mstate.cmatch = r_p.numpy(), c_p.numpy()
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng2.upload(gp, force=True)
            res = eng2.match_inplace(gp, mstate, shortest=shortest, kernel=kernel, improved=improved)
            e1.record(stream)
            e1.synchronize()
            if i >= args.warmup:
                ms_list.append(e0.elapsed_time(e1))
                parity_ok = parity_ok and (known is None or res == known)
        e_ms = statistics.mean(ms_list)

        # the same call sequence from PAGEABLE host arrays (plain numpy): what the C++ shim
        # (include/bmatch_b200.hpp, std::vector) and a ctypes caller pass; the library copies
        # them through its pinned staging ring
        pg_ms = []
        r_h, c_h = init.rmatch.copy(), init.cmatch.copy()
        for i in range(max(1, args.warmup // 2) + max(3, args.steps // 2)):
            r_h[:] = init.rmatch
            c_h[:] = init.cmatch
            mstate = bm.MatchingState.__new__(bm.MatchingState)
            mstate.rmatch, mstate.cmatch = r_h, c_h
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng2.upload(g, force=True)
            res = eng2.match_inplace(g, mstate, shortest=shortest, kernel=kernel, improved=improved)
            e1.record(stream)
            e1.synchronize()
            if i >= max(1, args.warmup // 2):
                pg_ms.append(e0.elapsed_time(e1))
                parity_ok = parity_ok and (known is None or res == known)

        # end to end with the GPU cheap initial matching (one-sided Karp-Sipser, then first-fit,
        # on the device inside the timed region): graph in, maximum matching out
        gi_ms = []
        for i in range(max(1, args.warmup // 2) + max(3, args.steps // 2)):
            mstate = bm.MatchingState.__new__(bm.MatchingState)
            mstate.rmatch, mstate.cmatch = r_p.numpy(), c_p.numpy()
            flush.fill_(1)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            eng2.upload(gp, force=True)
            res = eng2.match_inplace(gp, mstate, shortest=shortest, kernel=kernel, improved=improved,
                                     init_mode="gpu_ks")
            e1.record(stream)
            e1.synchronize()
            if i >= max(1, args.warmup // 2):
                gi_ms.append(e0.elapsed_time(e1))
                parity_ok = parity_ok and (known is None or res == known)
        gi_res = eng2.match(g, None, shortest=shortest, kernel=kernel, improved=improved, init_mode="gpu_ks")
        gi_kms, _ = eng2.last_kernel_time()
        if dist is not None:
            t = torch.tensor([e_ms, statistics.mean(pg_ms), statistics.mean(gi_ms)], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms, pg_mean, gi_mean = float(t[0]), float(t[1]), float(t[2])
        else:
            pg_mean, gi_mean = statistics.mean(pg_ms), statistics.mean(gi_ms)
        h2d = 8 * (g.nc + 1) + 4 * E + 4 * (g.nr + g.nc)
        d2h = 4 * (g.nr + g.nc)
        e2e = {"value": world * E / (e_ms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
               "host_buffers": "pinned (torch pin_memory)",
               # one-shot (upload + match per step): auto pulls only where one run repays the row index
               "pulled_dense_levels": args.bottom_up == "on" or (args.bottom_up == "auto" and auto_level == 2),
               "pageable": {"value": world * E / (pg_mean / 1e3), "ms_per_step": pg_mean,
                            "host_buffers": "pageable numpy arrays (the C++ shim's std::vector path)"},
               "gpu_init": {"value": world * E / (gi_mean / 1e3), "ms_per_step": gi_mean,
                            "h2d_bytes_per_step": 8 * (g.nc + 1) + 4 * E, "d2h_bytes_per_step": d2h,
                            "init": "BM_INIT_GPU_KS: degree-1 columns first, then first-fit, on the device",
                            "initial_cardinality": gi_res.counters.initial_cardinality,
                            "first_fit_cardinality": bm.cardinality(init),
                            "phases": gi_res.counters.outer_iterations, "kernel_ms": gi_kms,
                            "cardinality": bm.cardinality(gi_res.matching)}}
        parity_ok = parity_ok and (known is None or bm.cardinality(gi_res.matching) == known)
        del eng2

    # ---- roofline of the driver kernel (SURVEY.md §8d per-unit bytes) ----
    wr = 1 if kernel == bm.BfsKernel.GpubfsWr else 0
    c = counters
    nst = max(1, len(step_counters))

    def mean_of(attr):  # mean over the timed steps (phase counts differ from run to run)
        return sum(getattr(x, attr) for x in step_counters) / nst

    b_units = (12 * mean_of("edges_traversed") + (20 + 8 * wr) * mean_of("columns_scanned")
               + (8 + 4 * wr) * mean_of("columns_visited") + 20 * mean_of("walk_steps"))
    b_survey = b_units + mean_of("outer_iterations") * (12 * g.nc + 4 * g.nr + 4 * g.nr + 8 * g.nr + 8 * g.nc)
    peak, peak_src = measured_peak()
    achieved = b_units / (k_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"{args.config.lower()}_{args.algo}_ncu.json")
    if os.path.exists(prof):
        with open(prof) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    out = None
    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            res = cpu_reference_run(g, init)
            cpu = {"value": E / res["seconds"], "unit": "edges/s", "cores": res["cores"], "kind": res["kind"],
                   "sample": f"one full {args.config} run ({E} edges) of apfb-wr-ct "
                             f"{'parallel:' + str(res['cores']) if res['kind'] == 'reference' else 'serial port'}",
                   "seconds": res["seconds"], "cardinality": res["cardinality"]}
            parity_ok = parity_ok and res["cardinality"] == cards[-1]
        out = {
            "metric": METRIC, "value": world * E / (t_ms / 1e3), "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": data_kind(),
            "config": workload_config(args, g),
            "algorithm": f"{args.algo}-b200",
            "parallelism": "replicas" if world > 1 else "single-gpu",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "bm::driver_kernel (persistent, whole run)",
                         "algorithmic_bytes_per_launch": b_units, "survey_formula_bytes": b_survey,
                         "random_access_ceiling": random_access_ceiling(mean_of("edges_traversed"), k_ms)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "bottom_up": {"mode": args.bottom_up, "pulled_dense_levels": bool(pulled),
                          "row_index_ms": row_index_ms[-1] if row_index_ms else None,
                          # at >= 2^26 rows the upload builds the row index beside the copy, so
                          # bm_prepare_row_index finds it ready: its cost is inside upload_ms (and e2e)
                          "row_index_with_upload": bool(auto_level == 2),
                          "upload_ms": t_upload},
            "alternative": alt,
            "gpu_launches": launches,
            "clocks": sampler.summary(),
            "time_to_max_matching_ms": t_ms,
            "kernel_ms": k_ms,
            "teps": mean_of("edges_traversed") / (k_ms / 1e3),
            "cardinality": cards[-1],
            "parity": {"known_answer": known, "gpu_verify_violations": viol, "gpu_is_maximum": ismax,
                       "ok": bool(parity_ok)},
            "counters_mean": {k: mean_of(k) for k in ["outer_iterations", "columns_scanned", "edges_traversed",
                                                       "columns_visited", "walk_steps"]},
            "counters": {"outer_iterations": c.outer_iterations, "bfs_levels": c.bfs_launches_total(),
                         "columns_scanned": c.columns_scanned, "edges_traversed": c.edges_traversed,
                         "columns_visited": c.columns_visited, "walks": c.alternations_attempted,
                         "walk_steps": c.walk_steps, "fix_resets": c.fix_resets,
                         "serial_retries": c.serial_retries},
            "generation_s": t_gen, "timed_wall_s": wall,
        }
        emit(out)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="C5")
    ap.add_argument("--algo", choices=sorted(ALGOS), default="apfb-wr")
    ap.add_argument("--scale-div", type=int, default=1, help="shrink C2/C4/C5 by this factor (testing only)")
    ap.add_argument("--flush-mb", type=int, default=512)
    ap.add_argument("--ref-budget-s", type=float, default=180.0,
                    help="reference arm: wall budget for its timed full runs (a C5 run is ~1 min on 16 cores)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the other-direction measurement")
    ap.add_argument("--bottom-up", choices=["auto", "on", "off"], default="auto",
                    help="pull the dense BFS levels (direction-optimised; needs a row index, built on the first "
                         "run after an upload): auto = the engine decides per graph (BM_BU_AUTO)")
    ap.add_argument("--mode", choices=["auto", "single", "partition", "replicas"], default="auto",
                    help="auto: single GPU at N=1, column partition at N>1")
    ap.add_argument("--graph", default=None,
                    help="a Matrix Market (.mtx) or binary CSC (.bcsc) file to use instead of --config")
    args = ap.parse_args()
    if args.graph:
        global GRAPH_FILE
        GRAPH_FILE = os.path.abspath(args.graph)
        CONFIGS["file"] = f"{os.path.basename(args.graph)} (read by the parallel file reader, bmatch_b200_io.h)"
        args.config = "file"
    if args.warmup < 3 and args.impl == "b200":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        return run_reference_arm(args)
    world = dist_env()[0]
    if args.mode == "partition" or (args.mode == "auto" and world > 1):
        return run_partitioned(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
