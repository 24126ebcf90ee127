#!/usr/bin/env python3
"""bench.py -- checkpointed GB/s of the shadow-page sync hot path on B200.

A "step" is one coordinated checkpoint of the whole registered footprint:
A5 barrier -> A1 detect -> A2 compact -> A3 gather + commit (-> A4 copy-out for
the e2e figure) -> A5 all-reduce of the dirty/image bytes.  Before every step
the "application" rewrites a seeded d-fraction of the pages (synth writer
kernel) and L2 is scrubbed with a 256 MiB streaming read; both run outside the step's
CUDA events.  Inputs live in HBM (2 GiB > 126 MB L2 for C2).

  value  = F / T_dev : registered bytes per second with the image written to
           a device buffer (crum_checkpoint_gather_device), device-event time.
  e2e    = F / T_ckpt: same step through crum_checkpoint_gather into a pinned
           host image (D2H of the image inside the timed region).
  restore: F / T_restore through crum_restore_scatter (H2D inside).

Default workload (N=1): BASELINE.json configs[1] -- C2, one 1 GiB region,
64 KiB pages, 10% of pages rewritten per step, compare mode.

Multi-GPU: `python -m torch.distributed.run --nproc-per-node N bench.py --gpus N`
(one region set per rank, weak scaling, NCCL barrier + all-reduce only).
`--impl reference` times the CPU oracle (oracle/) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import signal
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "checkpointed GB/s (dirty detect+gather) at 1/2/4/8 B200; % of HBM roofline"
KiB, MiB, GiB = 1 << 10, 1 << 20, 1 << 30
FALLBACK_HBM_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="crum", choices=["crum", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="compare", choices=["compare", "hash", "tracked"])
    ap.add_argument("--page", type=int, default=64 * KiB)
    ap.add_argument("--dirty", type=float, default=None,
                    help="fraction of pages rewritten per step (default: 1%% for C1, 10%% otherwise, as BASELINE.json)")
    ap.add_argument("--region-gib", type=float, default=1.0)
    ap.add_argument("--compress", action="store_true", help="CRUM_COMPRESS gathers (DESIGN.md Z1-Z2)")
    ap.add_argument("--content", default="random", choices=["random", "half"],
                    help="half: the paper's 50%%-random vectors (PAPER.md:907-912): second half of every "
                         "region one repeated fp32 value; the writer then rewrites one word per dirty page")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the multi-rank path with several ranks sharing fewer GPUs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    a = ap.parse_args()
    if a.dirty is None:
        a.dirty = 0.01 if a.config == "c1" else 0.10
    return a


def workload(args, rank: int):
    """(specs, description).  specs: list of (nbytes, page_size, mode)."""
    mode = {"compare": 0, "hash": 1, "tracked": 2}[args.mode]
    if args.config == "c1":
        return [(4 * MiB, 4 * KiB, mode)], f"C1: one 4 MiB region, 4 KiB pages, {args.dirty:.0%} dirty, {args.mode}"
    if args.config == "c2":
        nb = int(args.region_gib * GiB)
        return [(nb, args.page, mode)], (f"C2: one {args.region_gib:g} GiB region, {args.page // KiB} KiB pages, "
                                         f"{args.dirty:.0%} dirty, {args.mode}")
    if args.config == "c3":
        sizes = synth.c3_region_sizes(20)
        return [(s, args.page, mode) for s in sizes], (f"C3: Rodinia-style 220 regions (15.96 GiB), "
                                                       f"{args.page // KiB} KiB pages, {args.dirty:.0%} dirty, {args.mode}")
    if args.config == "c5":
        # 240 GiB per GPU: 150 GiB of HBM regions + 90 GiB of host-resident
        # (UVA-mapped pinned) regions read over the host link; hash mode
        specs = [(75 * GiB, 2 * MiB, 1), (75 * GiB, 2 * MiB, 1), (45 * GiB, 2 * MiB, 1), (45 * GiB, 2 * MiB, 1)]
        return specs, "C5: 240 GiB per GPU (150 GiB HBM + 90 GiB host-resident), 2 MiB pages, 10% dirty, hash"
    big, small = synth.c4_region_sizes(synth.seed(4) + rank)
    specs = [(s, 64 * KiB, mode) for s in big] + [(s, 4 * KiB, mode) for s in small]
    return specs, f"C4: HPGMG-style 56 + 4096 regions (64.2 GiB) per GPU, 10% dirty, {args.mode}"


def host_resident(args):
    """Indices of the regions that live in host memory (config 5)."""
    return {2, 3} if args.config == "c5" else set()


def pin_to_gpu_node(node: int):
    """Run this rank's host threads on the CPUs of its GPU's NUMA node (the
    library also binds the pinned images there): the copy-out of SURVEY.md
    sec. 8(e) then stays on one socket.  No-op on single-node hosts (-1)."""
    if node < 0:
        return
    try:
        cpus = set()
        for part in open(f"/sys/devices/system/node/node{node}/cpulist").read().strip().split(","):
            a, _, b = part.partition("-")
            cpus.update(range(int(a), int(b or a) + 1))
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
    except (OSError, ValueError):
        pass


def read_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_traffic(key: str):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        return json.load(open(p)).get(key)
    except Exception:
        return None


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, gpu: int):
        self.path = f"/tmp/crum_clocks_{os.getpid()}.csv"
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                       "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.p.send_signal(signal.SIGTERM)
        self.p.wait()
        rows = []
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7 and f[0].isdigit():
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [int(r[0]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": int(rows[0][1]), "samples": len(rows),
                "reasons": reasons}


# ---------------------------------------------------------------------------
# CPU oracle (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------
def oracle_steps(specs, S, dirty, seconds: float, max_steps: int, min_steps: int = 1):
    """Time oracle checkpoint_gather on the same workload (host copies),
    writer outside the timing.  Returns (per-step seconds list, F, sample)."""
    from oracle import oracle
    o = oracle.Oracle()
    host = []
    for r, (nb, P, mode) in enumerate(specs):
        h = oracle.aligned_empty(nb)
        synth.fill_region(h, S, r)
        host.append(h)
        o.register(h, P, mode)
    cap = o.required_bytes()
    o.checkpoint_gather(capacity=cap)   # initial full image (epoch 0), untimed
    times = []
    t_start = time.perf_counter()
    epoch = 0
    while len(times) < max_steps and (len(times) < min_steps or time.perf_counter() - t_start < seconds):
        epoch += 1
        for r, (nb, P, mode) in enumerate(specs):
            pages = synth.choose_dirty(S, epoch, r, synth.n_pages(nb, P), dirty)
            synth.apply_writer(host[r], P, pages, S, epoch, r)
            if mode == 2:  # TRACKED: the writer marks what it writes
                o.mark_pages(r + 1, pages)
        t0 = time.perf_counter()
        st, img, rep = o.checkpoint_gather(capacity=cap)
        times.append(time.perf_counter() - t0)
        assert st == 0
    F = sum(nb for nb, _, _ in specs)
    return times, F


def oracle_steps_threads(specs, S, dirty, seconds: float, max_steps: int, threads: int):
    """The unmodified oracle on all host cores: the workload's pages are split
    into `threads` contiguous page-aligned slices, one oracle instance per
    slice and thread (the C oracle runs without the GIL); per step every
    thread applies its writer, a barrier, then the timed gathers, a barrier.
    Returns (per-step seconds list, F)."""
    import threading
    from oracle import oracle
    slices = [[] for _ in range(threads)]
    for r, (nb, P, mode) in enumerate(specs):
        n = synth.n_pages(nb, P)
        per = -(-n // threads)
        for t in range(threads):
            p0, p1 = t * per, min(n, (t + 1) * per)
            if p1 > p0:
                slices[t].append((r, p0 * P, min(nb, p1 * P) - p0 * P, P, mode))
    slices = [sl for sl in slices if sl]
    T = len(slices)
    bar = threading.Barrier(T)
    times, stop = [], [False]
    err = []

    def work(t):
        try:
            o = oracle.Oracle()
            host = []
            for k, (r, off, nb, P, mode) in enumerate(slices[t]):
                h = oracle.aligned_empty(nb)
                h[:] = synth.region_content(S, r, nb, off // 8)
                host.append(h)
                o.register(h, P, mode)
            cap = o.required_bytes()
            o.checkpoint_gather(capacity=cap)
            t_start = time.perf_counter()
            epoch = 0
            while True:
                epoch += 1
                for k, (r, off, nb, P, mode) in enumerate(slices[t]):
                    pages = synth.choose_dirty(S, epoch, (r << 8) + t, synth.n_pages(nb, P), dirty)
                    synth.apply_writer(host[k], P, pages, S, epoch, r)
                    if mode == 2:
                        o.mark_pages(k + 1, pages)
                bar.wait()
                t0 = time.perf_counter()
                st, _, _ = o.checkpoint_gather(capacity=cap)
                assert st == 0
                bar.wait()
                if t == 0:
                    times.append(time.perf_counter() - t0)
                    stop[0] = len(times) >= max_steps or time.perf_counter() - t_start > seconds
                bar.wait()
                if stop[0]:
                    return
        except Exception as e:  # surface in the caller
            err.append(e)
            bar.abort()

    ths = [threading.Thread(target=work, args=(t,)) for t in range(T)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    if err:
        raise err[0]
    return times, sum(nb for nb, _, _ in specs), T


def oracle_sample(specs, limit: int = 1 << 30):
    """The whole workload when it is at most ~2 GiB, else its first regions up
    to ~1 GiB (the last one truncated to whole pages): a bounded sample for
    the single-threaded CPU oracle, same shapes and page sizes."""
    F = sum(nb for nb, _, _ in specs)
    if F <= 2 * limit:
        return specs, "the same workload"
    out, acc = [], 0
    for nb, P, mode in specs:
        take = min(nb, max(P, (limit - acc) // P * P))
        out.append((take, P, mode))
        acc += take
        if acc >= limit:
            break
    return out, f"a {len(out)}-region slice of the workload"


def parity_check(args, ctx, crum, regions, specs, S, epoch, stream, dimg, cap, gflags, limit=4 << 30):
    """Untimed, after the measurements: copy the run's regions to the host,
    commit both sides (GPU sync_shadow; the oracle registers the copies and
    syncs), apply one more application epoch to both, then compare the GPU's
    device image with the oracle's image byte for byte -- the same launch
    configuration, page sizes and flags the timed steps used."""
    import torch
    F = sum(nb for nb, _, _ in specs)
    if F > limit:
        return {"checked": False, "why": f"footprint {F / GiB:g} GiB > {limit / GiB:g} GiB host-copy bound; "
                                         "tests/test_gpu_fullsize.py samples these sizes"}
    from oracle import oracle
    torch.cuda.synchronize()
    ctx.sync_shadow(stream)
    o = oracle.Oracle()
    host = []
    for r, (nb, P, mode) in enumerate(specs):
        h = oracle.aligned_empty(nb)
        h[:] = regions[r].cpu().numpy()
        host.append(h)
        o.register(h, P, mode)
    o.sync_shadow()
    half = args.content == "half"
    for r, (nb, P, mode) in enumerate(specs):
        pg = synth.choose_dirty(S, epoch, r, synth.n_pages(nb, P), args.dirty)
        synth.apply_writer(host[r], P, pg, S, epoch, r, touch=half)
        dp = torch.from_numpy(pg.astype(np.uint32)).to(regions[r].device)
        if mode == 2:
            o.mark_pages(r + 1, pg)
            crum.synth_write_pages_tracked(regions[r], nb, P, dp, dp.numel(), S, epoch, r,
                                           ctx.region_tracker(r + 1), stream=stream)
        else:
            crum.synth_write_pages(regions[r], nb, P, dp, dp.numel(), S, epoch, r, half, stream=stream)
    st, want, _ = o.checkpoint_gather(flags=oracle.COMPRESS if gflags & crum.COMPRESS else 0)
    rep = ctx.checkpoint_gather_device(dimg, cap, stream=stream, flags=gflags)
    torch.cuda.synchronize()
    got = dimg[:rep["image_bytes"]].cpu().numpy()
    ok = st == 0 and got.nbytes == want.nbytes and bool(np.array_equal(got, want))
    return {"checked": True, "ok": ok, "image_bytes": int(want.nbytes), "dirty_pages": int(rep["dirty_pages"]),
            "what": "one more epoch after the timed steps: GPU device image vs the oracle's image, "
                    "byte for byte (both sides committed to the run's state first)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    specs, desc = workload(args, 0)
    specs, what = oracle_sample(specs)
    S = synth.seed(1)
    steps = args.warmup + args.steps
    # the unmodified oracle on every host core: the sample is split into one
    # page slice per core, one oracle instance per thread (step = slowest)
    ncores = len(os.sched_getaffinity(0))
    times, F, T = oracle_steps_threads(specs, S, args.dirty, seconds=1e9, max_steps=steps, threads=ncores)
    t = times[args.warmup:]
    v = F / statistics.mean(t) / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(statistics.mean(t) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded splitmix64 words)",
            "config": {"workload": desc, "footprint_bytes": F},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": T, "kind": "oracle",
                             "sample": f"{what} ({F / GiB:g} GiB) split into {T} page slices, one oracle per "
                                       f"thread, {args.steps} timed steps (step = slowest thread)"},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import crum

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    pin_to_gpu_node(crum.device_numa_node(local))
    distributed = world > 1
    if distributed:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = torch.device("cuda", local)
    red_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")  # where collectives run
    stream = torch.cuda.Stream(device=dev)
    if args.config == "c5":
        args.mode = "hash"  # C5 is defined in hash mode
    specs, desc = workload(args, rank)
    S = synth.seed(1) + (rank << 20)
    F = sum(nb for nb, _, _ in specs)

    gflags = crum.COMPRESS if args.compress else 0
    if args.compress or args.content != "random":
        desc += f", content {args.content}" + (", compressed images" if args.compress else "")
    ctx = crum.Context(local, timing=True)
    regions = []
    with torch.cuda.stream(stream):
        for r, (nb, P, mode) in enumerate(specs):
            if r in host_resident(args):
                t = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
            else:
                t = torch.empty(nb, dtype=torch.uint8, device=dev)
            crum.synth_fill(t, nb, S, r, stream=stream)
            if args.content == "half":
                t[nb // 2 // 4 * 4:].view(torch.float32).fill_(0.25)
            regions.append(t)
            ctx.register_region(t, nb, P, mode)
    trackers = [ctx.region_tracker(r + 1) for r in range(len(specs))] if args.mode == "tracked" else None
    # the dirty pages of every epoch, precomputed on the host (untimed)
    n_epochs = args.warmup + args.steps + max(3, args.steps // 2) + max(4, args.steps // 2) + 2
    pages = [[torch.from_numpy(synth.choose_dirty(S, e, r, synth.n_pages(nb, P), args.dirty).astype(np.uint32)).to(dev)
              for r, (nb, P, _) in enumerate(specs)] for e in range(1, n_epochs + 1)]
    scrub = torch.empty(256 * MiB, dtype=torch.uint8, device=dev)
    # image capacity: a worst-case image when it fits beside the footprint
    # (asynchronous device path), else the exact bound for this dirty ratio
    # (the call then checks capacity itself and waits)
    worst = ctx.image_required_bytes()
    k_exp = sum(synth.dirty_count(args.dirty, synth.n_pages(nb, P)) for nb, P, _ in specs)
    free_b, _ = torch.cuda.mem_get_info(dev)
    cap = worst if worst + (1 << 30) < free_b - 2 * (1 << 30) and len(host_resident(args)) == 0 else \
        ctx.image_required_bytes(k_exp)
    async_ok = cap >= worst
    dimg = torch.empty(cap + 256, dtype=torch.uint8, device=dev)
    # epoch 0: the first (full) checkpoint, untimed
    ctx.sync_shadow(stream)   # epoch 0: commit the whole footprint (every page starts force-dirty)

    def app_epoch(e):
        for r, (nb, P, _) in enumerate(specs):
            pg = pages[e - 1][r]
            if trackers:
                # TRACKED: the application's writer marks what it writes (crum_device.h)
                crum.synth_write_pages_tracked(regions[r], nb, P, pg, pg.numel(), S, e, r, trackers[r],
                                               stream=stream)
            else:
                crum.synth_write_pages(regions[r], nb, P, pg, pg.numel(), S, e, r, args.content == "half",
                                       stream=stream)
        crum.synth_scrub(scrub, scrub.numel(), stream=stream)

    from paper_1808_00117_b200 import coord

    def coordinated(fn):
        """A5: barrier before detect; all-reduce of {dirty bytes, image bytes} after."""
        return coord.coordinated(fn).local

    def device_step():
        """One checkpoint into the device image, stream-asynchronous; with N > 1
        the coordinated all-reduce needs the totals, so the step waits for them."""
        if distributed:
            return coordinated(lambda: (ctx.checkpoint_gather_device(dimg, cap, stream=stream, flags=gflags,
                                                                     report=not async_ok),
                                        ctx.last_report())[1])
        ctx.checkpoint_gather_device(dimg, cap, stream=stream, flags=gflags, report=not async_ok)
        return None

    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    epoch = 0
    for _ in range(args.warmup):
        epoch += 1
        app_epoch(epoch)
        device_step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    clocks = Clocks(local)
    launches0 = ctx.launch_count
    t_wall0 = time.perf_counter()
    reps = []
    for i in range(args.steps):
        epoch += 1
        app_epoch(epoch)
        ev0[i].record(stream)
        device_step()
        ev1[i].record(stream)
        reps.append(ctx.last_report())  # after ev1: the wait is outside the timed interval
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    # context for fractions above 1.0: a plain streaming READ (no writes) of the
    # first HBM region, timed the same way; the denominator stays the measured copy
    dev_regs = [t for t in regions if t.is_cuda]
    rd_t = max(dev_regs + [scrub], key=lambda t: t.numel())  # the largest HBM buffer
    rd_n = min(rd_t.numel(), GiB) // 32 * 32
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    rd_ms = []
    for _ in range(5):
        e_a.record(stream)
        crum.synth_scrub(rd_t, rd_n, stream=stream)
        e_b.record(stream)
        e_b.synchronize()
        rd_ms.append(e_a.elapsed_time(e_b))
    read_stream = rd_n / (min(rd_ms) / 1e3) / 1e9
    # host-resident regions (config 5): the detect reads them over the host
    # link, so that link bounds the step; probe the SM-driven zero-copy read
    # of the same pinned memory, timed the same way
    host_regs = [t for t in regions if not t.is_cuda]
    host_link = None
    if host_regs:
        h_n = min(host_regs[0].numel(), 4 * GiB) // 32 * 32
        h_ms = []
        for _ in range(3):
            e_a.record(stream)
            crum.synth_scrub(host_regs[0], h_n, stream=stream)
            e_b.record(stream)
            e_b.synchronize()
            h_ms.append(e_a.elapsed_time(e_b))
        host_link = h_n / (min(h_ms) / 1e3) / 1e9
    launches = ctx.launch_count - launches0
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    T = sum(step_ms) / 1e3
    det_ms = [r["t_gather_ms"] if args.mode == "tracked" else r["t_detect_ms"] for r in reps]
    if distributed:
        t = torch.tensor([T, sum(det_ms)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        T, det_sum = float(t[0]), float(t[1])
    else:
        det_sum = sum(det_ms)
    value = world * F * args.steps / T / 1e9
    K = reps[-1]["dirty_pages"]
    KP = reps[-1]["image_bytes"]
    peak, peak_src = read_peaks()
    # dominant kernel.  Single-pass path (all compare, P <= 64 KiB): the fused
    # detect+compact+gather kernel, algorithmic bytes = read region + mirror
    # (2F) + write image payload + mirror (2 KP).  Otherwise A1 detect:
    # compare reads region + mirror (2F); hash reads region + table and writes
    # the new hashes (F + 16 N).
    n_pages = sum(synth.n_pages(nb, P) for nb, P, _ in specs)
    payload = reps[-1]["image_bytes"]
    fused = bool(reps[-1].get("path", 0) & 1)
    if fused:
        kname = "fused_compare"
        det_bytes = 2 * F + 2 * payload
    else:
        kname = "gather" if args.mode == "tracked" else f"detect_{args.mode}"
        det_bytes = {"compare": 2 * F, "hash": F + 16 * n_pages, "tracked": 2 * payload}[args.mode]
    det_t = det_sum / args.steps / 1e3
    achieved = det_bytes / det_t / 1e9
    # whole device phase: detect + gather reads/writes (compare also rewrites the
    # mirror of every listed page: + KP)
    dev_alg = {"compare": 2 * F + 3 * payload, "hash": F + 16 * n_pages + 2 * payload,
               "tracked": n_pages + 2 * payload}[args.mode]
    traffic_key = f"{kname}:{args.config}:{specs[0][1]}:{args.dirty}"
    in_bytes = {"compare": 2 * F, "hash": F + 8 * n_pages, "tracked": F}[args.mode]  # what one detect reads
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(T * 1e3 / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded splitmix64 words; seeded page choice per epoch)",
        "config": {"workload": desc, "footprint_bytes_per_gpu": F, "pages_per_gpu": n_pages,
                   "dirty_pages_per_step": K, "image_bytes_per_step": KP,
                   "l2": ((f"inputs {in_bytes / MiB:g} MiB (regions + shadow) > 126 MB L2; " if in_bytes > 126e6
                           else f"inputs {in_bytes / MiB:g} MiB (regions + shadow) fit in L2, so ") +
                          "a 256 MiB streaming read before every step evicts L2 (the writer's dirty lines are "
                          "written back there, untimed) and leaves it clean: every step starts cold"),
                   "timing": "per-step CUDA events around crum_checkpoint_gather_device on its stream; "
                             "application writer + scrub outside the events",
                   "wall_ms_per_step_incl_writer": round(wall * 1e3 / args.steps, 3),
                   "gpu_numa_node": crum.device_numa_node(local)},
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1),
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "alg_bytes_per_launch": det_bytes, "avg_launch_ms": round(det_t * 1e3, 4),
                     "traffic": read_traffic(traffic_key), "traffic_key": traffic_key,
                     "read_stream_GBs": round(read_stream, 1), "nominal_peak_GBs": 8000.0,
                     "note": "peak = measured copy (read+write); a read-only stream measured here reaches "
                             "read_stream_GBs, so read-dominated kernels can exceed frac 1.0"},
        "device_phase": {"alg_bytes_per_step": dev_alg, "achieved_GBs": round(dev_alg / (T / args.steps) / 1e9, 1),
                         "frac": round(dev_alg / (T / args.steps) / 1e9 / peak, 4)},
        "gpu_launches": launches,
        "gpu_launches_synth": 2 * args.steps * len(specs),
        "clocks": clk,
    }
    if host_link:
        # the detect's bytes that cross the host link, against the measured
        # zero-copy read of that link; the HBM figures stay beside them
        hb = sum(t.numel() for t in host_regs)
        hbm = line["roofline"]
        line["roofline"] = {"bound": "host_link", "kernel": kname, "achieved": round(hb / det_t / 1e9, 2),
                            "peak": round(host_link, 2), "unit": "GB/s",
                            "frac": round(hb / det_t / 1e9 / host_link, 4), "alg_bytes_per_launch": hb,
                            "avg_launch_ms": hbm["avg_launch_ms"], "traffic": None,
                            "peak_source": "SM-driven streaming read of the pinned host-resident region, "
                                           "timed in this run (the path the detect kernel reads it by)",
                            "note": f"{hb / GiB:g} GiB of the {F / GiB:g} GiB footprint are host-resident",
                            "hbm": hbm}
    if args.compress:
        line["compression"] = {"image_bytes": reps[-1]["image_bytes"], "dirty_bytes": reps[-1]["dirty_bytes"],
                               "ratio": round(reps[-1]["dirty_bytes"] / max(reps[-1]["image_bytes"], 1), 3),
                               "codec": "word-repeat (lag-2) unit codec, DESIGN.md Z1-Z2"}
    # ---- e2e: pinned host image, D2H inside the timed region ----
    if not args.no_e2e:
        img = ctx.new_image(cap)
        ctx.checkpoint_gather(img, stream=stream, flags=gflags)
        e2e_ms, e2e_reps = [], []
        for i in range(max(3, args.steps // 2)):
            epoch += 1
            app_epoch(epoch)
            torch.cuda.synchronize()
            if distributed:
                dist.barrier()
            t0 = time.perf_counter()
            e2e_reps.append(coordinated(lambda: ctx.checkpoint_gather(img, stream=stream, flags=gflags)))
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
        te = statistics.median(e2e_ms) / 1e3
        if distributed:
            t = torch.tensor([te], dtype=torch.float64, device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t[0])
        line["e2e"] = {"value": round(world * F / te / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                       "d2h_bytes_per_step": e2e_reps[-1]["image_bytes"], "ms_per_step": round(te * 1e3, 3),
                       "note": "crum_checkpoint_gather into pinned host memory, host wall clock per call "
                               "(median); the regions being checkpointed live in HBM by definition",
                       "image_numa_node": img.numa_node,
                       "link_GBs": (round(e2e_reps[-1]["image_bytes"] / e2e_reps[-1]["t_copy_ms"] / 1e6, 2)
                                    if e2e_reps[-1]["t_copy_ms"] > 0 else None)}
        # host-link roofline: a plain pinned D2H copy of the same size, timed live
        nb = max(min(e2e_reps[-1]["image_bytes"], 1 << 30), 1 << 20)
        hsrc = torch.empty(nb, dtype=torch.uint8, device=dev)
        hdst = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
        l_ms = []
        for _ in range(3):
            if distributed:
                dist.barrier()  # every rank copies at once: the concurrent (whole-box) link
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            with torch.cuda.stream(stream):
                hdst.copy_(hsrc, non_blocking=True)
            b_.record(stream)
            b_.synchronize()
            l_ms.append(a_.elapsed_time(b_))
        l_min = min(l_ms)
        if distributed:  # the slowest rank's concurrent copy sets the per-rank share
            t = torch.tensor([l_min], dtype=torch.float64, device=red_dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            l_min = float(t[0])
        link_peak = nb / (l_min / 1e3) / 1e9
        # the copy-out overlaps detection, so the e2e bound is the slower of the
        # link copy of the image and the device-only step
        e2e_ideal = world * F / max(e2e_reps[-1]["image_bytes"] / (link_peak * 1e9), T / args.steps)
        line["e2e"]["link_roofline"] = {"peak_GBs": round(link_peak, 2), "source": "pinned D2H copy of the "
                                        "image's size timed in this run (at N > 1: all ranks at once, the "
                                        "slowest rank's time)",
                                        "box_peak_GBs": round(world * link_peak, 2),
                                        "frac": round(line["e2e"]["value"] / (e2e_ideal / 1e9), 4),
                                        "ideal_value": round(e2e_ideal / 1e9, 1)}
        del hsrc, hdst
        # restore of the last image onto the live regions (H2D inside)
        r_ms = []
        for i in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rr = ctx.restore_scatter(img, stream=stream)
            r_ms.append((time.perf_counter() - t0) * 1e3)
        line["restore"] = {"value": round(F / (statistics.median(r_ms) / 1e3) / 1e9, 3), "unit": "GB/s",
                           "ms_per_call": round(statistics.median(r_ms), 3), "h2d_bytes": rr["image_bytes"],
                           "link_GBs": round(rr["image_bytes"] / (statistics.median(r_ms) / 1e3) / 1e9, 2)}
        # lazy restore (sec. 4.2 read-fault heuristic): time to first data and
        # per-fault latency for windows of 1, 2, 4, ... pages of region 1
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sess = ctx.restore_begin(img, stream=stream)
        begin_ms = (time.perf_counter() - t0) * 1e3
        n1 = synth.n_pages(specs[0][0], specs[0][1])
        faults, page = [], 0
        while page < n1 and len(faults) < 12:
            t0 = time.perf_counter()
            cov, res = sess.fetch(1, page, stream=stream)
            stream.synchronize()
            faults.append([cov, res, round((time.perf_counter() - t0) * 1e6, 1)])
            page += max(cov, 1)
        t0 = time.perf_counter()
        sess.end(stream=stream)
        line["lazy_restore"] = {"begin_ms": round(begin_ms, 3), "end_ms": round((time.perf_counter() - t0) * 1e3, 3),
                                "faults": faults,
                                "note": "sequential read faults on region 1 from page 0: [pages made present, "
                                        "image slots written, host wall us incl. stream sync]; zero-copy "
                                        "reads of the pinned image"}
        # forked checkpoint (sec. 3.3): the application pauses for
        # the gather only; a writer thread persists the image while the next epoch runs
        img2 = ctx.new_image(cap)
        tmpd = tempfile.mkdtemp(prefix="crum_bench_")
        pause_ms, w_ms = [], []
        try:
            for i in range(max(4, args.steps // 2)):
                epoch += 1
                app_epoch(epoch)
                torch.cuda.synchronize()
                im = (img, img2)[i % 2]
                im.persist_wait()
                t0 = time.perf_counter()
                ctx.checkpoint_gather(im, stream=stream, flags=gflags)
                pause_ms.append((time.perf_counter() - t0) * 1e3)
                im.persist(os.path.join(tmpd, f"r{rank}_{i % 2}.crum"))
            img.persist_wait()
            img2.persist_wait()
            t0 = time.perf_counter()
            img2.persist(os.path.join(tmpd, f"r{rank}_w.crum"))
            img2.persist_wait()
            w_ms.append((time.perf_counter() - t0) * 1e3)
        finally:
            shutil.rmtree(tmpd, ignore_errors=True)
        line["forked"] = {"pause_ms": round(statistics.median(pause_ms), 3),
                          "persist_GBs": round(img2.length / (w_ms[0] / 1e3) / 1e9, 3),
                          "persist_ms": round(w_ms[0], 3), "image_bytes": img2.length,
                          "note": "gather wall time with the previous image's writer in flight (two "
                                  "alternating pinned images); persist = one image written to "
                                  "tempfile.gettempdir() without fsync"}
        img2.destroy()
        img.destroy()
    # ---- cpu_baseline: the oracle on this workload, rank 0 at N=1 only ----
    if not args.no_cpu_baseline and world == 1:
        sample, what = oracle_sample(specs)
        times, Fo = oracle_steps(sample, synth.seed(1), args.dirty, seconds=args.cpu_seconds, max_steps=50)
        v = Fo / statistics.median(times) / 1e9
        line["cpu_baseline"] = {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                                "sample": f"{len(times)} oracle checkpoint_gather steps over {what} "
                                          f"({Fo / GiB:g} GiB, d={args.dirty}), writer untimed, median"}
        # context: the same oracle on every host core (independent page slices)
        ncores = len(os.sched_getaffinity(0))
        if ncores > 1:
            tt, Ft, T = oracle_steps_threads(sample, synth.seed(1), args.dirty, seconds=args.cpu_seconds,
                                             max_steps=50, threads=ncores)
            line["cpu_baseline"]["all_cores"] = {
                "value": round(Ft / statistics.median(tt) / 1e9, 4), "unit": "GB/s", "cores": T,
                "sample": f"{len(tt)} steps; the sample split into {T} page slices, one oracle per thread, "
                          f"writer untimed, step = slowest thread, median"}
    # ---- parity of this run's GPU result with the oracle ----
    if world == 1 and not host_resident(args):
        line["parity"] = parity_check(args, ctx, crum, regions, specs, S, epoch + 1, stream, dimg, cap, gflags)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
