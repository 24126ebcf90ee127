#!/usr/bin/env python3
"""bench.py -- checkpointed GB/s of the shadow-page sync hot path on B200.

A "step" is one coordinated checkpoint of the whole registered footprint:
A5 barrier -> A1 detect -> A2 compact -> A3 gather + commit -> A4 copy-out
into a pinned host image -> A5 all-reduce of the dirty/image bytes.  Before
every step the "application" rewrites a seeded d-fraction of the pages (synth
writer kernel) and L2 is scrubbed with a 256 MiB streaming read; both run
outside the step's CUDA events.  Inputs (the registered regions) live in HBM
when the timed region starts.

  value        = F / T_ckpt (registered bytes / (gather call ->
                 image complete in pinned host memory, commit done)); T_ckpt
                 from CUDA events on the call's stream, max over ranks.
  e2e          = the same call through the public Python API, host wall clock
                 per step including the A5 barrier + all-reduces (median).
  device_phase = the same step with the image written to an HBM buffer
                 (crum_checkpoint_gather_device): the HBM-roofline part.
  roofline     = the dominant kernel (A1 detect) of the device phase.
  restore      = F / T_restore through crum_restore_scatter (H2D inside).

Default workload (N=1): BASELINE.json's C4 per GPU -- 56 HPGMG-style level
vectors + 4096 box regions, 64.2 GiB, 10% of pages rewritten per step,
compare mode (the largest single-GPU config; C5 exceeds HBM).

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
    ap.add_argument("--config", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--mode", default="compare", choices=["compare", "hash", "tracked"])
    ap.add_argument("--page", type=int, default=64 * KiB)
    ap.add_argument("--dirty", type=float, default=None,
                    help="fraction of pages rewritten per step (default: 1%% for C1, 10%% otherwise, as BASELINE.json)")
    ap.add_argument("--region-gib", type=float, default=1.0)
    ap.add_argument("--compress", action="store_true",
                    help="CRUM_COMPRESS gathers: LZ77 + fixed-Huffman DEFLATE per 4 KiB unit (DESIGN.md Z2-Z3)")
    ap.add_argument("--content", default="random", choices=["random", "half", "hpgmg"],
                    help="half: the paper's 50%%-random vectors (PAPER.md:907-912): second half of every "
                         "region one repeated fp32 value; hpgmg: HPGMG-FV-like fp64 boxes (smooth fields, "
                         "constant coefficients, zero temporaries and ghost zones; synth.hpgmg_box_kinds); "
                         "for both the writer then rewrites one word per dirty page")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: test the multi-rank path with several ranks sharing fewer GPUs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fused", action="store_true",
                    help="CRUM_CFG_FUSED: the single-pass kernel for compare-only contexts of any size "
                         "(default: only up to 64 MiB)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--restore-full", action="store_true",
                    help="also time a FULL checkpoint (every page) into a pinned image and its restore onto the "
                         "live regions (SURVEY.md 8(d) C3 (a): full checkpoint + full restore)")
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
def oracle_steps(specs, S, dirty, seconds: float, max_steps: int, min_steps: int = 1, content: str = "random",
                 flags: int = 0):
    """Time oracle checkpoint_gather on the same workload (host copies),
    writer outside the timing.  Returns (per-step seconds list, F, sample)."""
    from oracle import oracle
    o = oracle.Oracle()
    host = []
    for r, (nb, P, mode) in enumerate(specs):
        h = oracle.aligned_empty(nb)
        synth.fill_region(h, S, r)
        if content == "half":
            h[nb // 2 // 4 * 4:].view(np.float32)[:] = 0.25
        elif content == "hpgmg":
            synth.hpgmg_fill(h, r)
        host.append(h)
        o.register(h, P, mode)
    cap = o.required_bytes()
    out = np.zeros(cap, dtype=np.uint8)  # reused: the timed step allocates nothing
    o.checkpoint_gather(flags=flags, capacity=cap, out=out)   # initial full image (epoch 0), untimed
    times = []
    t_start = time.perf_counter()
    epoch = 0
    while len(times) < max_steps and (len(times) < min_steps or time.perf_counter() - t_start < seconds):
        epoch += 1
        for r, (nb, P, mode) in enumerate(specs):
            pages = synth.choose_dirty(S, epoch, r, synth.n_pages(nb, P), dirty)
            synth.apply_writer(host[r], P, pages, S, epoch, r, touch=content != "random")
            if mode == 2:  # TRACKED: the writer marks what it writes
                o.mark_pages(r + 1, pages)
        t0 = time.perf_counter()
        st, img, rep = o.checkpoint_gather(flags=flags, capacity=cap, out=out)
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
            out = np.zeros(cap, dtype=np.uint8)
            o.checkpoint_gather(capacity=cap, out=out)
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
                st, _, _ = o.checkpoint_gather(capacity=cap, out=out)
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
    """A bounded sample of the workload for the CPU oracle, same shapes and
    page sizes: the whole workload when it is at most ~2 GiB; else every
    small region (< 1 MiB: C4's 4096 box regions) plus the leading regions up
    to ~`limit` bytes, the last one truncated to whole pages (SURVEY.md 8(d)
    oracle timing, step 4: "the first 1 GiB of large regions plus all 4096
    small regions")."""
    F = sum(nb for nb, _, _ in specs)
    if F <= 2 * limit:
        return specs, "the same workload"
    small = [(nb, P, m) for nb, P, m in specs if nb < MiB]
    out, acc = [], 0
    for nb, P, mode in specs:
        if nb < MiB:
            continue
        take = min(nb, max(P, (limit - acc) // P * P))
        out.append((take, P, mode))
        acc += take
        if acc >= limit:
            break
    what = f"a slice of the workload: the first {acc / GiB:g} GiB of its large regions"
    if small:
        what += f" plus all {len(small)} small regions (< 1 MiB)"
    return out + small, what


def host_info():
    """CPU model, logical CPUs usable, and the NUMA node(s) they sit on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    cpus = sorted(os.sched_getaffinity(0))
    nodes = []
    try:
        for d in sorted(os.listdir("/sys/devices/system/node")):
            if not (d.startswith("node") and d[4:].isdigit()):
                continue
            span = set()
            for part in open(f"/sys/devices/system/node/{d}/cpulist").read().strip().split(","):
                if part:
                    a, _, b = part.partition("-")
                    span.update(range(int(a), int(b or a) + 1))
            if span & set(cpus):
                nodes.append(int(d[4:]))
    except (OSError, ValueError):
        pass
    return {"cpu_model": model, "cpus": len(cpus), "numa_nodes": nodes}


def image_bytes_for(specs, dirty: float) -> int:
    """Image length of one step (format v1) from the seeded
    dirty counts -- config metadata shared by both arms, not a result."""
    R = len(specs)
    K = sum(synth.dirty_count(dirty, synth.n_pages(nb, P)) for nb, P, _ in specs)
    payload = sum(synth.dirty_count(dirty, synth.n_pages(nb, P)) * P for nb, P, _ in specs)
    poff = -(-(64 + 48 * R) // 4096) * 4096
    hashes = 8 * K if any(m == 1 for _, _, m in specs) else 0
    return poff + payload + -(-4 * K // 8) * 8 + hashes


def config_for(args, specs, desc, world: int):
    """The `config` object of the JSON line -- identical in both arms."""
    F = sum(nb for nb, _, _ in specs)
    N = sum(synth.n_pages(nb, P) for nb, P, _ in specs)
    K = sum(synth.dirty_count(args.dirty, synth.n_pages(nb, P)) for nb, P, _ in specs)
    in_bytes = {"compare": 2 * F, "hash": F + 8 * N, "tracked": F}[args.mode]
    return {"workload": desc, "config": args.config, "mode": args.mode, "dirty_fraction": args.dirty,
            "regions_per_gpu": len(specs), "page_sizes": sorted({P for _, P, _ in specs}),
            "footprint_bytes_per_gpu": F, "pages_per_gpu": N, "dirty_pages_per_step": K,
            "image_bytes_per_step": image_bytes_for(specs, args.dirty), "content": args.content,
            "compressed_images": bool(args.compress), "world_size": world,
            "l2": ((f"inputs {in_bytes / MiB:g} MiB (regions + shadow) > 126 MB L2; " if in_bytes > 126e6
                    else f"inputs {in_bytes / MiB:g} MiB (regions + shadow) fit in L2, so ") +
                   "a 256 MiB streaming read before every step evicts L2 (the writer's dirty lines are "
                   "written back there, untimed) and leaves it clean: every step starts cold")}


def hpgmg_fill_device(t, r: int):
    """HPGMG-FV-like content on the device (the paper's real-application image
    compresses 113 MB -> 14-16 MB): every 32 KiB box of fp64
    values is one of the kinds synth.hpgmg_box_kinds names -- a smooth field
    (solution / right-hand side), a constant coefficient (alpha, beta, Dinv)
    or zero (temporaries) -- with zero ghost layers at both ends of the box."""
    import torch
    n = t.numel() // 8
    nbox = n // 4096
    if nbox == 0:
        return
    kinds = synth.hpgmg_box_kinds(nbox, r)
    F = t[:nbox * 4096 * 8].view(torch.float64).view(nbox, 4096)
    x = torch.arange(4096, dtype=torch.float64, device=t.device)
    step = max(1, (256 << 20) // (4096 * 8))   # 256 MiB of boxes at a time (bounded temporaries)
    for b0 in range(0, nbox, step):
        b1 = min(nbox, b0 + step)
        k = torch.from_numpy(kinds[b0:b1]).to(t.device)
        blk = F[b0:b1]
        idx = torch.arange(b0, b1, dtype=torch.float64, device=t.device)
        smooth = torch.sin(x[None, :] * (0.001 + 0.0005 * (idx[:, None] % 7)) + idx[:, None]) * (1 + (idx[:, None] % 3))
        blk.copy_(torch.where((k <= 1)[:, None], smooth, blk))
        for kind, val in ((2, 1.0), (3, 1.0), (4, 1.0), (5, 1.0), (6, 1.0 / 6.0), (7, 0.0)):
            blk[k == kind] = val
        blk[:, :256] = 0
        blk[:, -256:] = 0


def snapshot_to_host(tensors):
    """Host copies of device tensors at HBM-footprint scale: the destination
    pages are first touched by all host threads at once (a single-threaded
    first touch of tens of GiB is what limits a plain .cpu()), then each
    tensor is copied through a pinned bounce buffer on one stream."""
    import torch
    from concurrent.futures import ThreadPoolExecutor
    outs = [np.empty(t.numel(), dtype=np.uint8) for t in tensors]
    jobs = []
    for a in outs:
        for o in range(0, a.size, 256 * MiB):
            jobs.append((a, o, min(a.size, o + 256 * MiB)))
    with ThreadPoolExecutor(max_workers=len(os.sched_getaffinity(0))) as ex:
        list(ex.map(lambda j: j[0][j[1]:j[2]].fill(0), jobs))
    chunk = 512 * MiB
    bounce = [torch.empty(chunk, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
    s = torch.cuda.Stream()
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    pending = [None, None]
    with ThreadPoolExecutor(max_workers=2) as ex:
        k = 0
        for t, a in zip(tensors, outs):
            src = t.reshape(-1)
            for o in range(0, a.size, chunk):
                n = min(chunk, a.size - o)
                b = k % 2
                if pending[b] is not None:
                    pending[b].result()       # the host copy out of this bounce buffer is done
                with torch.cuda.stream(s):
                    bounce[b][:n].copy_(src[o:o + n], non_blocking=True)
                    evs[b].record(s)
                evs[b].synchronize()
                pending[b] = ex.submit(np.copyto, a[o:o + n], bounce[b][:n].numpy())
                k += 1
        for f in pending:
            if f is not None:
                f.result()
    return outs


def parity_check(args, ctx, crum, regions, specs, rids, S, epoch, stream, img, dimg, cap, gflags):
    """Untimed, after the measurements, on every rank: commit the GPU side
    (sync_shadow), copy the committed regions to the host, run one more
    application epoch on the GPU and gather it THROUGH THE TIMED PATH (the
    pinned-image crum_checkpoint_gather, same image, capacity and flags).
    Every byte of that image is then checked against the CPU oracle region by
    region (tests/fullparity.py: a fresh oracle per region on the host copy,
    same writer epoch; header, table and padding rebuilt with struct + zlib),
    which works at any footprint.  Up to 4 GiB the device-image path
    (crum_checkpoint_gather_device) is also compared whole with the oracle's
    image after one more epoch."""
    import torch
    from oracle import oracle
    from tests import fullparity
    half = args.content != "random"   # the touch writer
    F = sum(nb for nb, _, _ in specs)
    if gflags and F > 4 * GiB:
        return {"checked": False, "why": "compressed images above 4 GiB: tests/test_gpu_compress.py"}
    torch.cuda.synchronize()
    ctx.sync_shadow(stream)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host = snapshot_to_host(regions)   # committed state, pageable host copies
    t_copy = time.perf_counter() - t0

    def write(e):
        for r, (nb, P, mode) in enumerate(specs):
            pg = synth.choose_dirty(S, e, r, synth.n_pages(nb, P), args.dirty)
            dp = torch.from_numpy(pg.astype(np.uint32)).to(regions[r].device)
            if mode == 2:
                crum.synth_write_pages_tracked(regions[r], nb, P, dp, dp.numel(), S, e, r,
                                               ctx.region_tracker(rids[r]), stream=stream)
            else:
                crum.synth_write_pages(regions[r], nb, P, dp, dp.numel(), S, e, r, half, stream=stream)

    write(epoch)
    ctx.checkpoint_gather(img, stream=stream, flags=gflags)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    if gflags:
        # compressed: the oracle gathers the same state with CRUM_COMPRESS (whole image)
        o = oracle.Oracle()
        for r, (nb, P, mode) in enumerate(specs):
            o.register(host[r], P, mode)
        o.sync_shadow()
        for r, (nb, P, mode) in enumerate(specs):
            pg = synth.choose_dirty(S, epoch, r, synth.n_pages(nb, P), args.dirty)
            synth.apply_writer(host[r], P, pg, S, epoch, r, touch=half)
            if mode == 2:
                o.mark_pages(r + 1, pg)
        st, want, _ = o.checkpoint_gather(flags=oracle.COMPRESS)
        got = img.view()
        ok = st == 0 and got.nbytes == want.nbytes and bool(np.array_equal(got, want))
        o.close()
        return {"checked": True, "ok": ok, "path": "crum_checkpoint_gather (pinned, compressed, as timed)",
                "image_bytes": int(got.nbytes), "oracle_s": round(time.perf_counter() - t1, 2),
                "what": "one more epoch after the timed steps: the GPU's compressed image vs the oracle's, byte "
                        "for byte"}
    res = fullparity.regionwise_check(img.view(), specs, rids, lambda r: host[r], S, epoch, args.dirty,
                                      touch=half, threads=min(16, len(os.sched_getaffinity(0))))
    out = {"checked": True, "ok": bool(res["ok"]), "path": "crum_checkpoint_gather (pinned image, as timed)",
           "image_bytes": res["image_bytes"], "checked_bytes": res["checked_bytes"],
           "dirty_pages": res["dirty_pages"], "oracle_s": round(time.perf_counter() - t1, 2),
           "host_copy_s": round(t_copy, 2),
           "what": "one more epoch after the timed steps; every byte of the GPU image checked against the CPU "
                   "oracle region by region (tests/fullparity.py), header/table/padding via struct + zlib"}
    F = sum(nb for nb, _, _ in specs)
    if F <= 4 * GiB and dimg is not None:
        # the device-image path too: state after `epoch` is committed on both
        o = oracle.Oracle()
        for r, (nb, P, mode) in enumerate(specs):
            fullparity_state = host[r]  # regionwise_check applied epoch `epoch` to it in place
            o.register(fullparity_state, P, mode)
        o.sync_shadow()
        e2 = epoch + 1
        for r, (nb, P, mode) in enumerate(specs):
            pg = synth.choose_dirty(S, e2, r, synth.n_pages(nb, P), args.dirty)
            synth.apply_writer(host[r], P, pg, S, e2, r, touch=half)
            if mode == 2:
                o.mark_pages(r + 1, pg)
        write(e2)
        st, want, _ = o.checkpoint_gather()
        rep = ctx.checkpoint_gather_device(dimg, cap, stream=stream, flags=gflags)
        torch.cuda.synchronize()
        got = dimg[:rep["image_bytes"]].cpu().numpy()
        out["device_path_ok"] = bool(st == 0 and got.nbytes == want.nbytes and np.array_equal(got, want))
        out["ok"] = out["ok"] and out["device_path_ok"]
        o.close()
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config == "c5":
        args.mode = "hash"
    specs, desc = workload(args, 0)
    config = config_for(args, specs, desc, world)
    sample, what = oracle_sample(specs)
    S = synth.seed(1)
    steps = args.warmup + args.steps
    # the unmodified oracle on every host core: the sample is split into one
    # page slice per core, one oracle instance per thread (step = slowest)
    ncores = len(os.sched_getaffinity(0))
    times, Fs, T = oracle_steps_threads(sample, S, args.dirty, seconds=1e9, max_steps=steps, threads=ncores)
    t = times[args.warmup:]
    v = Fs / statistics.mean(t) / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(statistics.mean(t) * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (seeded splitmix64 words; seeded page choice per epoch)",
            "config": config,
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": T, "kind": "oracle",
                             "sample": f"{what} ({Fs / GiB:g} GiB) split into {T} page slices, one oracle per "
                                       f"thread, {args.steps} timed steps (step = slowest thread); GB/s of "
                                       f"sampled footprint", **host_info()},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def timed_read_stream(crum, buf, nbytes, stream, reps=5):
    import torch
    e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(reps):
        e_a.record(stream)
        crum.synth_scrub(buf, nbytes, stream=stream)
        e_b.record(stream)
        e_b.synchronize()
        ms.append(e_a.elapsed_time(e_b))
    return nbytes / (min(ms) / 1e3) / 1e9


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    import __graft_entry__
    __graft_entry__.build()
    from paper_1808_00117_b200 import coord, crum

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
        world = dist.get_world_size()
    dev = torch.device("cuda", local)
    red_dev = dev if args.dist_backend == "nccl" else torch.device("cpu")  # where collectives run
    stream = torch.cuda.Stream(device=dev)
    if args.config == "c5":
        args.mode = "hash"  # C5 is defined in hash mode
    specs, desc = workload(args, rank)
    S = synth.seed(1) + (rank << 20)
    F = sum(nb for nb, _, _ in specs)
    n_pages = sum(synth.n_pages(nb, P) for nb, P, _ in specs)

    gflags = crum.COMPRESS if args.compress else 0
    if args.compress or args.content != "random":
        desc += f", content {args.content}" + (", compressed images" if args.compress else "")
    t_setup = time.perf_counter()
    ctx = crum.Context(local, timing=True, flags=crum.CFG_FUSED if args.fused else 0)
    regions = []
    with torch.cuda.stream(stream):
        for r, (nb, P, mode) in enumerate(specs):
            if r in host_resident(args):
                t = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
            else:
                t = torch.empty(nb, dtype=torch.uint8, device=dev)
            regions.append(t)
        # one launch for every region's seeded content (C4: 4152 regions)
        crum.synth_fill_regions([(t, nb, r) for r, (t, (nb, _, _)) in enumerate(zip(regions, specs))], S,
                                stream=stream)
        for r, (t, (nb, P, mode)) in enumerate(zip(regions, specs)):
            if args.content == "half":
                t[nb // 2 // 4 * 4:].view(torch.float32).fill_(0.25)
            elif args.content == "hpgmg":
                hpgmg_fill_device(t, r)
    stream.synchronize()
    t_alloc = time.perf_counter() - t_setup
    # one batch registration (crum_register_regions): one descriptor rebuild
    rids = ctx.register_regions([(t, nb, P, mode) for t, (nb, P, mode) in zip(regions, specs)])
    t_reg = time.perf_counter() - t_setup - t_alloc
    trackers = [ctx.region_tracker(rid) for rid in rids] if args.mode == "tracked" else None
    # the dirty pages of an epoch: chosen on the host (seeded recipe), one H2D
    # copy per epoch, sliced per region
    page_cache = {}

    def pages_of(e):
        if e not in page_cache:
            lists = [synth.choose_dirty(S, e, r, synth.n_pages(nb, P), args.dirty).astype(np.uint32)
                     for r, (nb, P, _) in enumerate(specs)]
            flat = torch.from_numpy(np.concatenate(lists) if lists else np.zeros(0, np.uint32)).to(dev)
            out, o = [], 0
            for a in lists:
                out.append(flat[o:o + a.size])
                o += a.size
            page_cache.clear()
            page_cache[e] = out
        return page_cache[e]

    scrub = torch.empty(256 * MiB, dtype=torch.uint8, device=dev)
    k_exp = sum(synth.dirty_count(args.dirty, synth.n_pages(nb, P)) for nb, P, _ in specs)
    # the pinned image: a worst-case image when that is small (<= 2 GiB: the
    # gather commits as it streams; C1 takes the one-launch small path), else
    # the exact bound for this dirty ratio (the gather streams range by range
    # and commits once the image is known to fit)
    worst_img = ctx.image_required_bytes()
    cap = worst_img if worst_img <= 2 * GiB else ctx.image_required_bytes(k_exp)
    img = ctx.new_image(cap)
    ctx.sync_shadow(stream)   # epoch 0: commit the whole footprint (every page starts force-dirty)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t_setup
    print(f"[bench] setup {setup_s:.1f} s: allocate + fill {t_alloc:.1f} s, register {len(specs)} regions "
          f"{t_reg:.1f} s", file=sys.stderr, flush=True)

    def app_epoch(e, scrub_l2=True):
        pg_e = pages_of(e)
        if trackers:
            for r, (nb, P, _) in enumerate(specs):
                # TRACKED: the application's writer marks what it writes (crum_device.h)
                crum.synth_write_pages_tracked(regions[r], nb, P, pg_e[r], pg_e[r].numel(), S, e, r, trackers[r],
                                               stream=stream)
        else:
            # every region's writer in one launch (C4: 4152 regions)
            crum.synth_write_regions([(regions[r], nb, P, r, pg_e[r], pg_e[r].numel())
                                      for r, (nb, P, _) in enumerate(specs)], S, e, args.content != "random",
                                     stream=stream)
        if scrub_l2:
            crum.synth_scrub(scrub, scrub.numel(), stream=stream)

    epoch = 0

    # ---- headline: checkpoint into the pinned host image (A1-A5) ----
    def pinned_step():
        g = coord.coordinated(lambda: ctx.checkpoint_gather(img, stream=stream, flags=gflags))
        return g

    for _ in range(args.warmup):
        epoch += 1
        app_epoch(epoch)
        pinned_step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    clocks = Clocks(local)
    launches0 = ctx.launch_count
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    wall_ms, greps = [], []
    for i in range(args.steps):
        epoch += 1
        app_epoch(epoch)
        # the application's writes + L2 scrub finish before the call: the host
        # clock (e2e) then times the call alone, as the events do
        stream.synchronize()
        ev0[i].record(stream)
        t0 = time.perf_counter()
        greps.append(pinned_step())
        wall_ms.append((time.perf_counter() - t0) * 1e3)
        ev1[i].record(stream)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    launches = ctx.launch_count - launches0
    step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    T = coord.max_over_ranks(sum(step_ms) / 1e3)
    value = world * F * args.steps / T / 1e9
    rep = greps[-1].local
    KP = rep["image_bytes"]
    K = rep["dirty_pages"]
    # slot bytes of the step (sum of P over the listed pages) from the image length
    poff = -(-(64 + 48 * len(specs)) // 4096) * 4096
    slot_bytes = KP - poff - (-(-4 * K // 8) * 8) - (8 * K if any(m == 1 for _, _, m in specs) else 0)
    te = coord.max_over_ranks(statistics.median(wall_ms) / 1e3)
    copy_ms = statistics.median([g.local["t_copy_ms"] for g in greps])

    # host-link roofline: a plain pinned D2H copy of the image's size, timed live
    nb = max(min(KP, 1 << 30), 1 << 20)
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
    link_peak = nb / (coord.max_over_ranks(min(l_ms)) / 1e3) / 1e9
    del hsrc, hdst

    # ---- device phase: the same step with the image in HBM ----
    worst = ctx.image_required_bytes()
    free_b, _ = torch.cuda.mem_get_info(dev)
    dcap = worst if worst + (1 << 30) < free_b - 2 * (1 << 30) and not host_resident(args) else cap
    async_ok = dcap >= worst
    dimg = torch.empty(dcap + 256, dtype=torch.uint8, device=dev)

    def device_step():
        if distributed:
            return coord.coordinated(lambda: (ctx.checkpoint_gather_device(dimg, dcap, stream=stream, flags=gflags,
                                                                           report=not async_ok),
                                              ctx.last_report())[1])
        ctx.checkpoint_gather_device(dimg, dcap, stream=stream, flags=gflags, report=not async_ok)
        return None

    for _ in range(args.warmup):
        epoch += 1
        app_epoch(epoch)
        device_step()
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    d0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    d1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    dreps = []
    for i in range(args.steps):
        epoch += 1
        app_epoch(epoch)
        d0[i].record(stream)
        device_step()
        d1[i].record(stream)
        dreps.append(ctx.last_report())  # after d1: the wait is outside the timed interval
    torch.cuda.synchronize()
    call_latency = None
    if F <= 64 * MiB:
        # small footprints are latency-bound: per call cold (the device phase
        # above: the writer + an L2 scrub before every call) and warm (the
        # writer only, so the region and its mirror may still sit in L2)
        w0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        w1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for i in range(args.steps):
            epoch += 1
            app_epoch(epoch, scrub_l2=False)
            w0[i].record(stream)
            device_step()
            w1[i].record(stream)
        torch.cuda.synchronize()
        call_latency = {
            "cold_us": round(statistics.median(a.elapsed_time(b) for a, b in zip(d0, d1)) * 1e3, 2),
            "warm_us": round(statistics.median(a.elapsed_time(b) for a, b in zip(w0, w1)) * 1e3, 2),
            "kernel_us": round(statistics.median(r["t_detect_ms"] for r in dreps) * 1e3, 2),
            "note": "device image; CUDA events on the call's stream around each call, median over the steps; "
                    "cold = writer + L2 scrub before each call, warm = writer only; kernel = the checkpoint "
                    "kernel(s) alone (the report's t_detect_ms)"}
    if distributed:
        dist.barrier()
    clk = clocks.stop()
    Td = coord.max_over_ranks(sum(a.elapsed_time(b) for a, b in zip(d0, d1)) / 1e3) / args.steps
    det_ms = [r["t_gather_ms"] if args.mode == "tracked" else r["t_detect_ms"] for r in dreps]
    det_t = coord.max_over_ranks(sum(det_ms) / args.steps) / 1e3
    dpay = dreps[-1]["image_bytes"]
    peak, peak_src = read_peaks()
    fused = bool(dreps[-1].get("path", 0) & 1)
    small_path = bool(dreps[-1].get("path", 0) & 4)
    # algorithmic bytes: what the method must move, not what a
    # staged implementation moves.  Dominant kernel: A1 detect -- compare reads
    # region + mirror (2F); hash reads region + table, writes new hashes
    # (F + 16N); tracked: the gather (reads + writes the listed pages).
    if fused:
        # a single-pass kernel (one launch: detect + compaction + gather + commit)
        kname = "small_ckpt" if small_path else "single_pass"
        det_bytes = {"compare": 2 * F + 2 * slot_bytes, "tracked": n_pages + 2 * slot_bytes}.get(args.mode, 0)
        det_ms = [r["t_detect_ms"] for r in dreps]
        det_t = coord.max_over_ranks(sum(det_ms) / args.steps) / 1e3
    else:
        kname = "gather" if args.mode == "tracked" else f"detect_{args.mode}"
        det_bytes = {"compare": 2 * F, "hash": F + 16 * n_pages, "tracked": 2 * slot_bytes}[args.mode]
    achieved = det_bytes / det_t / 1e9
    # device phase, algorithmic: compare 2F + 2KP (read region + mirror, write
    # mirror + image); hash F + 8N + 8K + KP; tracked N + 2KP
    dev_alg = {"compare": 2 * F + 2 * slot_bytes, "hash": F + 8 * n_pages + 8 * K + slot_bytes,
               "tracked": n_pages + 2 * slot_bytes}[args.mode]
    # context for fractions above 1.0: a plain streaming READ of the largest HBM
    # buffer -- at least 2 GiB (a temporary buffer when every region is smaller:
    # a short read stream under-measures the rate, C3's 256 MiB gave 5.8 TB/s)
    dev_regs = [t for t in regions if t.is_cuda]
    rd_t = max(dev_regs + [scrub], key=lambda t: t.numel())
    if rd_t.numel() < 2 * GiB:
        free_b, _ = torch.cuda.mem_get_info(dev)
        if free_b > 4 * GiB:
            rd_t = torch.zeros(2 * GiB, dtype=torch.uint8, device=dev)
    read_stream = timed_read_stream(crum, rd_t, min(rd_t.numel(), 8 * GiB) // 32 * 32, stream)
    del rd_t
    host_regs = [t for t in regions if not t.is_cuda]
    host_link = None
    if host_regs:
        host_link = timed_read_stream(crum, host_regs[0], min(host_regs[0].numel(), 4 * GiB) // 32 * 32, stream, 3)

    config = config_for(args, specs, desc, world)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(T * 1e3 / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (seeded splitmix64 words; seeded page choice per epoch)",
        "config": config,
        "timing": {"value": "per-step CUDA events on the call's stream around the coordinated "
                            "crum_checkpoint_gather into a pinned host image (returns when the image is "
                            "complete and committed); application writer + L2 scrub outside the events; "
                            "sum over the K steps, max over ranks",
                   "setup_s": round(setup_s, 2),
                   "comm": {"backend": dist.get_backend() if distributed else None, "ranks": world}},
        "step": {"bound": "host_link", "image_bytes": KP, "dirty_pages": K, "t_copy_ms": round(copy_ms, 3),
                 "link_peak_GBs": round(link_peak, 2),
                 "link_peak_source": "pinned D2H copy of the image's size timed in this run (N > 1: all ranks "
                                     "at once, the slowest rank)",
                 "ideal_ms": round(max(KP / (link_peak * 1e9), Td) * 1e3, 3),
                 "frac": round(max(KP / (link_peak * 1e9), Td) / (T / args.steps), 4),
                 "note": "the step's bound is the copy-out of the image over the host link (or the device "
                         "phase if longer); frac = ideal / measured step"},
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1),
                     "peak": peak, "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "alg_bytes_per_launch": det_bytes, "avg_launch_ms": round(det_t * 1e3, 4),
                     "traffic": read_traffic(f"{kname}:{args.config}:{specs[0][1]}:{args.dirty}"),
                     "read_stream_GBs": round(read_stream, 1), "nominal_peak_GBs": 8000.0,
                     "measured_in": ("the device phase's timed steps: the one-launch small kernel's own globaltimer "
                                     "stamps (first CTA in -> last CTA out; CUDA events around it would add their "
                                     "own cost to a ~15 us kernel), inside the CUDA-event-timed step"
                                     if small_path else
                                     "the device phase's timed steps (CUDA events around the kernel on its stream)"),
                     "note": "peak = measured copy (read+write); a read-only stream measured here reaches "
                             "read_stream_GBs, so read-dominated kernels can exceed frac 1.0"},
        "device_phase": {"value": round(world * F / Td / 1e9, 3), "unit": "GB/s", "ms_per_step": round(Td * 1e3, 4),
                         "alg_bytes_per_step": dev_alg, "achieved_GBs": round(dev_alg / Td / 1e9, 1),
                         "frac": round(dev_alg / Td / 1e9 / peak, 4),
                         "what": "crum_checkpoint_gather_device (image in HBM), CUDA events; algorithmic "
                                 "bytes compare 2F+2KP, hash F+8N+8K+KP, tracked N+2KP"},
        "e2e": {"value": round(world * F / te / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": KP, "ms_per_step": round(te * 1e3, 3),
                "note": "the public Python API (Context.checkpoint_gather under coord.coordinated), host wall "
                        "clock per step incl. the A5 barrier + all-reduces, median, max over ranks; the "
                        "regions being checkpointed live in HBM by definition",
                "image_numa_node": img.numa_node},
        "call_latency": call_latency,
        "gpu_launches": launches,
        # the application's writer (one batched launch; TRACKED: one per region) + the L2 scrub,
        # enqueued before each step's events (not in the timed interval)
        "gpu_launches_synth": args.steps * ((len(specs) if args.mode == "tracked" else 1) + 1),
        "clocks": clk,
    }
    if host_link:
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
        line["compression"] = {"image_bytes": rep["image_bytes"], "dirty_bytes": rep["dirty_bytes"],
                               "ratio": round(rep["dirty_bytes"] / max(rep["image_bytes"], 1), 3),
                               "detect_to_last_chunk_packed_ms": round(
                                   statistics.median([g.local["t_gather_ms"] for g in greps]), 3),
                               "codec": "per 4 KiB unit: greedy LZ77 (12-bit hash, every position inserted) in "
                                        "one fixed-Huffman DEFLATE block, zero units empty, incompressible units "
                                        "raw (DESIGN.md Z2-Z3)"}
    # ---- restore of the last timed step's image onto the live regions (H2D inside) ----
    torch.cuda.synchronize()
    r_ms = []
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rr = ctx.restore_scatter(img, stream=stream)
        r_ms.append((time.perf_counter() - t0) * 1e3)
    tr = statistics.median(r_ms) / 1e3
    line["restore"] = {"value": round(F / tr / 1e9, 3), "unit": "GB/s", "ms_per_call": round(tr * 1e3, 3),
                       "h2d_bytes": rr["image_bytes"], "link_GBs": round(rr["image_bytes"] / tr / 1e9, 2),
                       "link_frac": round(rr["image_bytes"] / tr / 1e9 / link_peak, 4),
                       "note": "link_frac against the run's pinned D2H probe (H2D measured 55.6 vs D2H 55.2 GB/s "
                               "on the pool's boxes, profiles/r01/probe_box.json)"}
    if args.restore_full:
        # C3 (a): a FULL checkpoint (every page, CRUM_FULL) and its restore,
        # both through the pinned image (host link in both directions)
        fimg = ctx.new_image(ctx.image_required_bytes())
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fr = ctx.checkpoint_gather(fimg, stream=stream, flags=crum.FULL)
        tg = time.perf_counter() - t0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rr2 = ctx.restore_scatter(fimg, stream=stream)
        trf = time.perf_counter() - t0
        line["restore_full"] = {"image_bytes": fr["image_bytes"], "checkpoint_GBs": round(F / tg / 1e9, 3),
                                "checkpoint_ms": round(tg * 1e3, 3), "restore_GBs": round(F / trf / 1e9, 3),
                                "restore_ms": round(trf * 1e3, 3),
                                "checkpoint_link_frac": round(fr["image_bytes"] / tg / 1e9 / link_peak, 4),
                                "restore_link_frac": round(rr2["image_bytes"] / trf / 1e9 / link_peak, 4),
                                "note": "CRUM_FULL gather into a pinned image and crum_restore_scatter of it onto "
                                        "the live regions, host wall clock, one call each"}
        fimg.destroy()
    # lazy restore (sec. 4.2 read-fault heuristic): per-fault latency for
    # windows of 1, 2, 4, ... pages of region 1
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sess = ctx.restore_begin(img, stream=stream)
    begin_ms = (time.perf_counter() - t0) * 1e3
    n1 = synth.n_pages(specs[0][0], specs[0][1])
    faults, page = [], 0
    while page < n1 and len(faults) < 12:
        t0 = time.perf_counter()
        cov, res = sess.fetch(rids[0], page, stream=stream)
        stream.synchronize()
        faults.append([cov, res, round((time.perf_counter() - t0) * 1e6, 1)])
        page += max(cov, 1)
    t0 = time.perf_counter()
    sess.end(stream=stream)
    line["lazy_restore"] = {"begin_ms": round(begin_ms, 3), "end_ms": round((time.perf_counter() - t0) * 1e3, 3),
                            "faults": faults,
                            "note": "sequential read faults on region 1 from page 0: [pages made present, "
                                    "image slots written, host wall us incl. stream sync]; zero-copy reads of "
                                    "the pinned image"}
    # forked checkpoint (sec. 3.3): the application pauses for
    # the gather only; a writer thread persists the image (fsync'd) while the
    # next epoch runs
    if KP <= 2 * GiB and not args.no_e2e:
        img2 = ctx.new_image(cap)
        tmpd = tempfile.mkdtemp(prefix="crum_bench_")
        pause_ms = []
        # O_DIRECT + fsync (storage, not the page cache) where the filesystem allows it
        direct = True
        try:
            img.persist(os.path.join(tmpd, "probe.crum"), fsync=True, direct=True)
            img.persist_wait()
        except crum.CrumError:
            direct = False
        try:
            for i in range(4):
                epoch += 1
                app_epoch(epoch)
                torch.cuda.synchronize()
                im = (img, img2)[i % 2]
                im.persist_wait()
                t0 = time.perf_counter()
                ctx.checkpoint_gather(im, stream=stream, flags=gflags)
                pause_ms.append((time.perf_counter() - t0) * 1e3)
                im.persist(os.path.join(tmpd, f"r{rank}_{i % 2}.crum"), fsync=True, direct=direct)
            img.persist_wait()
            img2.persist_wait()
            t0 = time.perf_counter()
            img2.persist(os.path.join(tmpd, f"r{rank}_w.crum"), fsync=True, direct=direct)
            img2.persist_wait()
            w_ms = (time.perf_counter() - t0) * 1e3
        finally:
            shutil.rmtree(tmpd, ignore_errors=True)
        line["forked"] = {"pause_ms": round(statistics.median(pause_ms), 3),
                          "persist_GBs": round(img2.length / (w_ms / 1e3) / 1e9, 3), "persist_ms": round(w_ms, 3),
                          "image_bytes": img2.length,
                          "note": "gather wall time with the previous image's writer in flight (two alternating "
                                  "pinned images); persist = one image written and fsync'd to "
                                  "tempfile.gettempdir()" + (" with O_DIRECT (no page-cache copy)" if direct else
                                                             " (buffered: the filesystem refused O_DIRECT)"),
                          "o_direct": direct}
        img2.destroy()
    # ---- cpu_baseline: the oracle on a bounded sample, rank 0 at N=1 only ----
    if not args.no_cpu_baseline and world == 1:
        sample, what = oracle_sample(specs)
        times, Fo = oracle_steps(sample, synth.seed(1), args.dirty, seconds=args.cpu_seconds, max_steps=50,
                                 content=args.content, flags=4 if args.compress else 0)
        v = Fo / statistics.median(times) / 1e9
        line["cpu_baseline"] = {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                                "sample": f"{len(times)} oracle checkpoint_gather steps over {what} "
                                          f"({Fo / GiB:g} GiB, d={args.dirty}), writer untimed, median; GB/s of "
                                          f"sampled footprint", **host_info()}
        ncores = len(os.sched_getaffinity(0))
        if ncores > 1:
            tt, Ft, Tn = oracle_steps_threads(sample, synth.seed(1), args.dirty, seconds=args.cpu_seconds,
                                              max_steps=50, threads=ncores)
            line["cpu_baseline"]["all_cores"] = {
                "value": round(Ft / statistics.median(tt) / 1e9, 4), "unit": "GB/s", "cores": Tn,
                "sample": f"{len(tt)} steps; the sample split into {Tn} page slices, one oracle per thread, "
                          f"writer untimed, step = slowest thread, median"}
    # ---- parity of this run's GPU result with the oracle, on every rank ----
    if not host_resident(args):
        par = parity_check(args, ctx, crum, regions, specs, rids, S, epoch + 1, stream, img,
                           dimg if F <= 4 * GiB else None, dcap, gflags)
        if distributed:
            allp = [None] * world
            dist.all_gather_object(allp, {"rank": rank, "ok": par.get("ok"), "checked": par.get("checked"),
                                          "checked_bytes": par.get("checked_bytes")})
            par["ranks"] = allp
            par["ok"] = all(p["ok"] for p in allp) if par.get("checked") else par.get("ok")
        line["parity"] = par
    else:
        line["parity"] = {"checked": False, "why": "host-resident regions: tests/test_gpu_fullsize.py samples C5"}
    img.destroy()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
