"""Benchmark: word16 32-lane interleaved rANS round trip on B200.

Workload (BASELINE.json configs[1]): 256 MiB of
synthetic Zipf(s=1.1) bytes per GPU, N=32 lanes, 16-bit word renorm,
64 KiB chunks (4096 independent streams), scale_bits 12. One STEP is the
whole path over that batch, inputs resident in HBM:

    histogram -> [NCCL all-reduce of 256 x u64 when N>1] -> quantize + tables
    -> chunked encode -> ICH1 directory (word-offset scan) -> chunked decode
       straight from the encoder's slot layout

The packed ICH1 payload is built when the stream leaves HBM (the e2e leg
packs it straight into pinned host memory); its in-HBM cost is reported
as "pack".

value = raw bytes of all ranks / step time (GB/s = 1e9 B/s), max over
ranks. Inputs (256 MiB) exceed the 126 MB L2, so no explicit flush.
Decode and encode GB/s are also reported separately (per-phase CUDA events
on the launching stream). `e2e` is the same round trip through the public
HostCodec API from pinned host memory (H2D + D2H inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

`--impl reference` times the unmodified reference (oracle/_ref: ilans with
its compiled Cython kernels) on the host cores, fork pool over all cores,
on a bounded sample of the same chunks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MIB = 1 << 20
METRIC = "rANS decode & encode GB/s per B200 and 8xB200; compression ratio vs entropy"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mib", type=int, default=256, help="MiB per GPU")
    ap.add_argument("--chunk", type=int, default=64 * 1024)
    ap.add_argument("--lanes", type=int, default=32)
    ap.add_argument("--scale-bits", type=int, default=12)
    ap.add_argument("--zipf-s", type=float, default=1.1)
    ap.add_argument("--seed", type=int, default=1234)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-plugin", action="store_true")
    ap.add_argument("--plugin-only", action="store_true",
                    help="only the plugin_e2e leg (threads 1,2,4,8,16)")
    ap.add_argument("--sweep", action="store_true", help="config 4: entropy x precision sweep")
    ap.add_argument("--stress", action="store_true",
                    help="config 5: small chunks x many streams (framing / tail overhead)")
    ap.add_argument("--global-mib", type=int, default=0,
                    help="config 3: fixed global size split over the ranks (strong scaling)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    return ap.parse_args()


def hbm_peak():
    """HBM roofline denominator: the driver-written MEASURED_PEAKS.json (a
    coder kernel is timed alone, so a burst figure when one is given, else
    the plain HBM figure), else the profiling recipe's 6.65 TB/s fallback."""
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            peaks = json.loads(f.read_text())
        except ValueError:
            peaks = {}
        flat = {}

        def walk(d, pre=""):
            for k, v in d.items():
                if isinstance(v, dict):
                    walk(v, pre + k + ".")
                elif isinstance(v, (int, float)):
                    flat[pre + k] = float(v)
        walk(peaks)
        hbm = {k: v for k, v in flat.items() if "hbm" in k.lower()}
        for pref in ("burst", "hbm_gbs", ""):
            hit = [k for k in sorted(hbm) if pref in k.lower()]
            if hit:
                return hbm[hit[0]], f"measured (MEASURED_PEAKS.json {hit[0]})"
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def config_of(a, world):
    if a.global_mib:
        per = a.global_mib * MIB / world
        name = (f"config3: {a.global_mib} MiB global synthetic Zipf(s={a.zipf_s}) bytes split "
                f"over {world} GPU(s) (strong scaling)")
        glob = a.global_mib * MIB
    else:
        per = a.mib * MIB
        name = f"config2: {a.mib} MiB/GPU synthetic Zipf(s={a.zipf_s}) bytes"
        glob = a.mib * MIB * world
    return {
        "workload": f"{name}, N={a.lanes} lanes word16, {a.chunk // 1024} KiB chunks, "
                    f"sb={a.scale_bits}, round trip (model build + encode + ICH1 directory + "
                    f"decode)",
        "bytes_per_gpu": int(per),
        "global_bytes": glob,
        "chunk_len": a.chunk,
        "lanes": a.lanes,
        "scale_bits": a.scale_bits,
        "zipf_s": a.zipf_s,
        "seed": a.seed,
        "parallelism": f"chunk-sharded x{world} ({'strong' if a.global_mib else 'weak'}), "
                       "histogram all-reduce" if world > 1 else "single GPU",
        "l2": f"inputs ({per / MIB:.0f} MiB/GPU) vs the 126 MB L2: "
              + ("larger, no flush needed" if per > 126e6 else "SMALLER: L2-resident"),
    }


# ---------------------------------------------------------------- clocks ---
REASONS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


class Clocks:
    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/ilans_clocks_{os.getpid()}.csv")

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def wait_lines(self, k: int, timeout: float = 5.0) -> None:
        """Block until the sampler has written k more lines (so short timed
        regions are still bracketed by samples)."""
        if self.proc is None:
            return
        def count():
            try:
                return self.path.read_text().count("\n")
            except OSError:
                return 0
        start = count()
        t0 = time.time()
        while count() < start + k and time.time() - t0 < timeout:
            time.sleep(0.02)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm, mx, active = [], [], set()
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(REASONS, parts[2:6]):
                if v.lower().startswith("active"):
                    active.add(name)
        self.path.unlink(missing_ok=True)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(active), "samples": len(sm)}


# --------------------------------------------------------- CPU reference ---
def _ref_hist_worker(args):
    """Fork-pool worker: np.bincount of a contiguous byte range (the
    reference's model-build call site, cli._build_table / bench._table_for,
    split over the pool); returns (seconds, counts)."""
    lo, hi = args
    msg = _REF_STATE[0]
    t0 = time.perf_counter()
    counts = np.bincount(msg[lo:hi], minlength=256)
    return time.perf_counter() - t0, counts


def _ref_worker(args):
    """Fork-pool worker: round-trip a contiguous range of chunks with the
    reference ext kernels on fork-inherited data; returns (seconds, ok)."""
    lo, hi = args
    from ilans.interleave import decode_interleaved, encode_interleaved
    from ilans.rans import WORD16

    msg, table, C, lanes = _REF_STATE
    t0 = time.perf_counter()
    ok = True
    for k in range(lo, hi):
        chunk = msg[k * C:(k + 1) * C]
        c = encode_interleaved(chunk, table, lanes, WORD16, backend="ext")
        out = decode_interleaved(c, backend="ext")
        ok &= bool(np.array_equal(out, chunk))
    return time.perf_counter() - t0, ok


_REF_STATE = None


def cpu_reference(msg: np.ndarray, sb: int, C: int, lanes: int, per_core_mib: int = 16):
    """Time the reference CPU path on a bounded sample of the same workload,
    on a fork pool over all host cores (per_core_mib per core):

    1. model build -- np.bincount of each worker's byte range (the
       reference's call site, cli._build_table, split over the pool), summed,
       then SymbolTable.from_counts (one thread);
    2. an encode + decode round trip of every sampled chunk with the
       reference ext kernels (reference bench.py:86-93 per chunk).

    ``value`` covers both; ``coding_only_GBps`` is step 2 alone and
    ``single_thread_model_build_s`` is the reference's own unsplit bincount."""
    global _REF_STATE
    import multiprocessing as mp

    ref_dir = ROOT / "oracle" / "_ref"
    kind = "reference"
    if (ref_dir / "ilans" / "__init__.py").exists():
        sys.path.insert(0, str(ref_dir))
        os.environ["ILANS_BACKEND"] = "ext"
        from ilans import backend as ref_backend
        from ilans.rans import SymbolTable as RefTable

        if ref_backend.EXT is None:
            kind = "port"
    else:
        kind = "port"
    cores = len(os.sched_getaffinity(0))
    chunks_per_core = max(1, (per_core_mib * MIB) // C)
    total_chunks = len(msg) // C
    n_chunks = min(total_chunks, chunks_per_core * cores)
    if kind != "reference":
        n_chunks = min(total_chunks, chunks_per_core)
    sample_msg = msg[: n_chunks * C]
    sample = n_chunks * C
    t0 = time.perf_counter()
    np.bincount(sample_msg, minlength=int(sample_msg.max()) + 1)
    t_model_1t = time.perf_counter() - t0
    if kind == "reference":
        ctx = mp.get_context("fork")
        _REF_STATE = (sample_msg, None, C, lanes)
        bounds = np.linspace(0, sample, cores + 1).astype(np.int64)
        with ctx.Pool(cores) as pool:
            hres = pool.map(_ref_hist_worker, [(int(bounds[i]), int(bounds[i + 1]))
                                               for i in range(cores)])
        t0 = time.perf_counter()
        counts = np.sum([h[1] for h in hres], axis=0)
        counts = counts[: int(np.nonzero(counts)[0][-1]) + 1]
        table = RefTable.from_counts(counts.tolist(), sb)
        t_model = max(h[0] for h in hres) + time.perf_counter() - t0
        _REF_STATE = (msg, table, C, lanes)
        ranges = np.array_split(np.arange(n_chunks), cores)
        jobs = [(int(r[0]), int(r[-1]) + 1) for r in ranges if len(r)]
        t0 = time.perf_counter()
        with ctx.Pool(len(jobs)) as pool:
            res = pool.map(_ref_worker, jobs)
        wall = time.perf_counter() - t0
        busy = max(r[0] for r in res)
        ok = all(r[1] for r in res)
        workers = len(jobs)
        per_core = statistics.median((hi - lo) * C / r[0] / 1e9 for (lo, hi), r in zip(jobs, res))
    else:  # oracle port (C restatement), single core
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle

        t0 = time.perf_counter()
        counts = np.bincount(sample_msg, minlength=int(sample_msg.max()) + 1)
        freqs_s = oracle.quantize(counts, sb)
        f, cum, slot = oracle.table_views(freqs_s, sb)
        t_model = time.perf_counter() - t0
        t0 = time.perf_counter()
        ok = True
        for k in range(n_chunks):
            chunk = msg[k * C:(k + 1) * C]
            p, s = oracle.encode_interleaved_u16(chunk, f, cum, sb, lanes)
            out, _ = oracle.decode_interleaved_u16(p, s, slot, f, cum, sb, len(chunk), lanes)
            ok &= bool(np.array_equal(out, chunk))
        wall = busy = time.perf_counter() - t0
        workers = 1
        per_core = n_chunks * C / busy / 1e9
    return {
        "value": sample / (t_model + busy) / 1e9,
        "unit": "GB/s",
        "cores": workers,
        "kind": kind,
        "sample": f"{n_chunks} x {C // 1024} KiB chunks ({sample / MIB:.0f} MiB) of the same "
                  f"workload: model build (np.bincount split over {workers} workers + "
                  f"SymbolTable.from_counts, {t_model:.3f}s) then encode+decode round trip per "
                  f"chunk with the reference "
                  f"{'ext backend' if kind == 'reference' else 'C port'} on {workers} "
                  f"worker(s) (slowest worker {busy:.3f}s; wall incl. fork {wall:.2f}s)",
        "round_trip_ok": ok,
        "coding_only_GBps": sample / busy / 1e9,
        "model_build_s": t_model,
        "single_thread_model_build_s": t_model_1t,
        "single_core_round_trip_GBps": per_core,
        "wall_s": wall,
    }


# ---------------------------------------------------------------- b200 ---
def fused_consumer(codec, d_out, n, dev, reps=5):
    """decode fused with its consumer. The consumer here is a
    per-chunk Adler-32 (zlib-compatible): fused, the decoder hands each
    decoded block to it in registers; unfused, the decoder writes the bytes
    to HBM and a second kernel reads them back."""
    import torch

    fused = codec.decode_adler32(n, slots=True).clone()
    codec.decode_slots(d_out, n)
    if not torch.equal(fused, codec.adler32(d_out, n)):
        raise SystemExit("fused decode+adler32 mismatch")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize(dev)
    ev[0].record()
    for _ in range(reps):
        codec.decode_adler32(n, slots=True)
    ev[1].record()
    for _ in range(reps):
        codec.decode_slots(d_out, n)
        codec.adler32(d_out, n)
    ev[2].record()
    torch.cuda.synchronize(dev)
    f_ms, u_ms = ev[0].elapsed_time(ev[1]) / reps, ev[1].elapsed_time(ev[2]) / reps
    return {"consumer": "per-chunk Adler-32 of the decoded bytes",
            "fused_GBps": n / (f_ms * 1e-3) / 1e9, "fused_ms": f_ms,
            "unfused_GBps": n / (u_ms * 1e-3) / 1e9, "unfused_ms": u_ms,
            "hbm_bytes_avoided": 2 * n}


_PLUGIN = None


def _plugin_range(job):
    """The reference's per-chunk loop (reference bench.py:86-93 shape, the
    _ref_worker below) over chunks [lo, hi), through the reference kernel
    boundary Backend("b200") with host buffers; returns (seconds, ok)."""
    from paper_1402_3392_b200.interleave import decode_interleaved, encode_interleaved
    from paper_1402_3392_b200.rans import WORD16

    lo, hi = job
    msg, table, C, lanes = _PLUGIN
    outs = []
    t0 = time.perf_counter()
    for k in range(lo, hi):
        chunk = msg[k * C:(k + 1) * C]
        c = encode_interleaved(chunk, table, lanes, WORD16, backend="b200")
        outs.append(decode_interleaved(c, backend="b200"))
    el = time.perf_counter() - t0
    # round-trip check after the clock (the reference bench verifies
    # outside its timed region too, reference bench.py:86-93)
    ok = all(np.array_equal(o, msg[k * C:(k + 1) * C]) for k, o in zip(range(lo, hi), outs))
    return el, ok


CONFIG1_DIGEST = "1ea63c4d860a4650"  # byte8 N=2 sb=12 container


def config1(ref: bool, repeats: int = 3):
    """BASELINE config 1: byte8 (8-bit digits, L = 2^23), N = 2 lanes, sb =
    12, 1 MiB of Zipf(1.1) bytes -- the reference's scalar path
    (interleave.py:155-179). Input: default_rng(1).choice, the BASELINE.md
    section 3 known-answer input, so the container digest is checked too.
    ref=True times the unmodified reference (oracle/_ref, pure Python);
    otherwise the single-stream drop-in call on the B200 (one warp, 2 lanes)."""
    import hashlib

    if ref:
        sys.path.insert(0, str(ROOT / "oracle" / "_ref"))
        from ilans.interleave import decode_interleaved, encode_interleaved
        from ilans.rans import BYTE8, SymbolTable
    else:
        from paper_1402_3392_b200.interleave import decode_interleaved, encode_interleaved
        from paper_1402_3392_b200.rans import BYTE8, SymbolTable
    p = (np.arange(256) + 1.0) ** -1.1
    msg = np.random.default_rng(1).choice(256, 1 << 20, p=p / p.sum()).astype(np.uint8)
    table = SymbolTable.from_counts(np.bincount(msg, minlength=int(msg.max()) + 1).tolist(), 12)
    enc, dec = [], []
    for _ in range(1 if ref else repeats):
        t0 = time.perf_counter()
        c = encode_interleaved(msg, table, 2, BYTE8)
        t1 = time.perf_counter()
        out = decode_interleaved(c)
        t2 = time.perf_counter()
        enc.append(t1 - t0)
        dec.append(t2 - t1)
    digest = hashlib.sha256(c.to_bytes()).hexdigest()[:16]
    return {"workload": "config1: byte8 N=2 sb=12, 1 MiB Zipf(1.1) (default_rng(1).choice), "
                        "one container", "impl": "reference pure-Python scalar path" if ref
            else "B200 single-stream drop-in (one warp, 2 lanes)",
            "encode_MBps": len(msg) / min(enc) / 1e6, "decode_MBps": len(msg) / min(dec) / 1e6,
            "round_trip_MBps": len(msg) / (min(enc) + min(dec)) / 1e6,
            "container_sha256_16": digest, "digest_ok": digest == CONFIG1_DIGEST,
            "round_trip_ok": bool(np.array_equal(out, msg))}


def plugin_e2e(msg_h, table, C, N, threads_list=(1, 8, 16), sample_mib=256):
    """SURVEY 8b drop-in path: the reference's per-chunk loop
    (encode_interleaved + decode_interleaved per 64 KiB chunk, one Container
    each) through Backend("b200") -- one warp per call, host buffers in and
    out, every call synchronous -- on T host threads (ctypes releases the
    GIL during each call; the library keeps one stream, staging buffer and
    cached model per thread, so T calls are in flight at once). Each thread
    warms its own context up first; the clock runs from a barrier to the
    last thread's end."""
    global _PLUGIN
    import threading

    k = min(len(msg_h) // C, (sample_mib * MIB) // C)
    _PLUGIN = (msg_h, table, C, N)
    rows = {}
    for T in threads_list:
        ranges = [r for r in np.array_split(np.arange(k), T) if len(r)]
        bar = threading.Barrier(len(ranges) + 1)
        res = [None] * len(ranges)

        def worker(i, r):
            _plugin_range((int(r[0]), int(r[0]) + min(2, len(r))))  # context + model warm-up
            bar.wait()
            res[i] = _plugin_range((int(r[0]), int(r[-1]) + 1))
            bar.wait()

        ths = [threading.Thread(target=worker, args=(i, r)) for i, r in enumerate(ranges)]
        for t in ths:
            t.start()
        bar.wait()
        t0 = time.perf_counter()
        bar.wait()
        wall = time.perf_counter() - t0
        for t in ths:
            t.join()
        if not all(r[1] for r in res):
            raise SystemExit("plugin round-trip mismatch")
        rows[f"threads_{T}"] = {"GBps": k * C / wall / 1e9, "s": wall,
                                "us_per_chunk_round_trip": 1e6 * wall * len(ranges) / k}
    return {"what": f"reference per-chunk loop through Backend('b200'): {k} x {C // 1024} KiB "
                    f"chunks, encode_interleaved + decode_interleaved (one Container per chunk, "
                    f"N={N}), host numpy buffers, wall clock", **rows}


def e2e(a, n, k_chunks, C, N, sb, dev, d_msg, allreduce, world, global_bytes, slots=3):
    """The same round trip through the public host API (chunked.HostCodec)
    from pinned host memory: every step uploads its message, builds the
    model, encodes, downloads the framed payload, uploads it again, decodes
    and downloads the decoded bytes. Steps are pipelined two deep through
    encode_async / decode_async (step i+1's upload overlaps step i's
    downloads: PCIe is full duplex); the blocking encode() + decode() form is
    timed too ("sequential")."""
    import torch
    import torch.distributed as dist

    from paper_1402_3392_b200.chunked import HostCodec

    hc = HostCodec(n, C, N, sb, dev, counts_allreduce=allreduce, slots=slots,
                   batch_bytes=64 << 20)
    h_msg = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_msg.copy_(d_msg[:n])
    h_outs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]

    def round_trip(i):
        ej = hc.encode_async(h_msg, n)
        dj = hc.decode_async(ej, h_outs[i % 2])
        return ej, dj

    for i in range(3):  # warm-up + round-trip gate through every slot
        round_trip(i)[1].wait()
        if not torch.equal(h_outs[i % 2], h_msg):
            raise SystemExit("e2e round-trip mismatch")
    # the bench's K steps (capped): pipeline fill and drain amortise as in a
    # real stream of messages (4 steps 22.1 GB/s, 8: 24.3, 16: 25.2, 64: 26.3)
    steps = max(4, min(a.steps, 64))

    def timed(run):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        h2d, d2h = run()
        torch.cuda.synchronize(dev)
        el = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(el, op=dist.ReduceOp.MAX)
        return global_bytes * steps / float(el.item()) / 1e9, h2d // steps, d2h // steps

    def pipelined():
        # message i+1 is queued before round trip i's decode, so its upload
        # fills the link while encode i's first payload batch comes down
        h2d = d2h = 0
        pending = []
        ejs = [hc.encode_async(h_msg, n)]
        for i in range(steps):
            if i + 1 < steps:
                ejs.append(hc.encode_async(h_msg, n))
            dj = hc.decode_async(ejs[i], h_outs[i % 2])
            h2d += ejs[i].h2d_bytes + dj.h2d_bytes
            d2h += ejs[i].d2h_bytes + dj.d2h_bytes
            pending.append(dj)
            if len(pending) == 2:
                pending.pop(0).wait()  # step i-1's decoded bytes are on the host
        for dj in pending:
            dj.wait()
        return h2d, d2h

    def sequential():
        h2d = d2h = 0
        for _ in range(steps):
            p, o, s = hc.encode(h_msg, n)
            h2d += hc.h2d_bytes; d2h += hc.d2h_bytes
            hc.decode(p, o, s, n, h_outs[0])
            h2d += hc.h2d_bytes; d2h += hc.d2h_bytes
        return h2d, d2h

    v, h2d, d2h = timed(pipelined)
    if not (torch.equal(h_outs[0], h_msg) and torch.equal(h_outs[1], h_msg)):
        raise SystemExit("e2e round-trip mismatch")
    vs, _, _ = timed(sequential)
    return {"value": v, "unit": "GB/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "chunked.HostCodec encode_async()+decode_async() from pinned host memory, "
                   f"up to {slots} round trips in flight",
            "sequential_GBps": vs, "steps": steps,
            "timing": "wall clock around synchronized steps, max over ranks"}


def run_b200(a):
    import torch
    import torch.distributed as dist

    from paper_1402_3392_b200 import _lib
    from paper_1402_3392_b200.chunked import DeviceCodec, HostCodec, n_chunks_for
    from paper_1402_3392_b200.synth import synth_device, zipf_probs, entropy_bits

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        print(f"bench.py: WORLD_SIZE={world} but --gpus {a.gpus}; using WORLD_SIZE",
              file=sys.stderr)
    # one process per GPU; --dist-backend gloo (+ wrap-around device index)
    # only exists to smoke-test the multi-rank logic on a single-GPU box
    local = local % max(1, torch.cuda.device_count()) if a.dist_backend == "gloo" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if a.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    from paper_1402_3392_b200.dist import allreduce_counts, shard_for

    C, N, sb = a.chunk, a.lanes, a.scale_bits
    # weak scaling: the global message is world x mib MiB; this rank owns a
    # contiguous chunk-aligned shard of it (dist.shard_for)
    # (--global-mib: strong scaling, the global message is fixed, config 3)
    global_bytes = a.global_mib * MIB if a.global_mib else a.mib * MIB * world
    shard = shard_for(global_bytes, rank, world, C)
    n = shard.n_bytes
    k_chunks = n_chunks_for(n, C)

    d_msg = synth_device(n, a.zipf_s, a.seed, first=shard.byte_lo, device=dev)
    d_out = torch.empty(n, dtype=torch.uint8, device=dev)
    codec = DeviceCodec(n, C, N, sb, dev)
    stream = torch.cuda.current_stream(dev)

    def allreduce(counts):
        allreduce_counts(counts)  # NCCL all-reduce of 256 x u64 (int64 sum == u64 sum)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # One step: model build, encode, the ICH1 directory (word offsets) and a
    # decode straight from the encoder's slot layout. The packed ICH1 payload
    # is built only when the stream leaves HBM (e2e packs into pinned host
    # memory); its in-HBM cost is timed separately below ("pack").
    side = torch.cuda.Stream(dev)

    def directory_beside_decode():
        # the directory only feeds the ICH1 framing: it runs on a side
        # stream next to the decode (which reads the slot layout)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            codec.directory(n)
        codec.decode_slots(d_out, n)
        stream.wait_stream(side)

    def step(marks=None):
        if marks: marks[0].record(stream)
        codec.histogram(d_msg, n)
        allreduce(codec.counts)
        codec.build_table_from_counts()
        if marks: marks[1].record(stream)
        codec.encode(d_msg, n, frame=False)
        if marks: marks[2].record(stream)
        if marks: marks[3].record(stream)
        directory_beside_decode()
        if marks: marks[4].record(stream)

    # round-trip gate before timing (reference bench.py:92-93)
    codec.reset_status()
    step()
    codec.check_status()
    torch.cuda.synchronize(dev)
    if not torch.equal(d_out, d_msg[:n]):
        raise SystemExit("bench round-trip mismatch")
    consumed = codec.consumed[:k_chunks]
    offs = codec.offsets[: k_chunks + 1]
    if not torch.equal(consumed, offs[1:] - offs[:-1]):
        raise SystemExit("decoder did not consume every payload word")
    total_words = int(offs[-1])
    # the packed stream decodes to the same bytes (and is what ICH1 carries)
    codec.frame_range(n, 0, k_chunks, codec.payload.data_ptr())
    codec.decode(d_out, n)
    codec.check_status()
    torch.cuda.synchronize(dev)
    if not torch.equal(d_out, d_msg[:n]) or not torch.equal(codec.consumed[:k_chunks], consumed):
        raise SystemExit("packed-stream round-trip mismatch")
    for _ in range(max(0, a.warmup - 1)):
        step()
    torch.cuda.synchronize(dev)

    # 1) eager steps with per-phase events (the phase breakdown)
    marks = [[ev() for _ in range(5)] for _ in range(a.steps)]
    l0 = _lib.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = ev(); t1 = ev()
    t0.record(stream)
    for i in range(a.steps):
        step(marks[i])
    t1.record(stream)
    torch.cuda.synchronize(dev)
    launches_per_step = (_lib.launch_count() - l0) // a.steps
    eager_ms = t0.elapsed_time(t1)
    phase = np.array([[m[j].elapsed_time(m[j + 1]) for j in range(4)] for m in marks])

    # 2) the headline: the same step captured once as a CUDA graph and
    #    replayed (no per-kernel launch gaps); eager under torchrun, where the
    #    step contains the NCCL all-reduce
    #    (under torchrun the NCCL all-reduce stays eager between two graphs:
    #    histogram | all-reduce | model + encode + framing + decode)
    def part_a():
        codec.histogram(d_msg, n)

    def part_b():
        codec.build_table_from_counts()
        codec.encode(d_msg, n, frame=False)
        directory_beside_decode()

    def capture(fn):
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            fn()
        stream.wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    graph = None
    try:
        if world == 1:
            g = capture(step)
            graph = g.replay
        else:
            ga, gb = capture(part_a), capture(part_b)

            def graph():
                ga.replay()
                allreduce(codec.counts)
                gb.replay()
        graph()
        torch.cuda.synchronize(dev)
        if not torch.equal(d_out, d_msg[:n]):
            raise SystemExit("bench round-trip mismatch (graph)")
    except RuntimeError as e:  # capture unsupported: time eagerly
        print(f"graph capture failed, timing eager steps: {e}", file=sys.stderr)
        graph = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with Clocks(local) as clk:
        clk.wait_lines(1)
        t0 = ev(); t1 = ev()
        t0.record(stream)
        for i in range(a.steps):
            if graph is not None:
                graph()
            else:
                step()
        t1.record(stream)
        torch.cuda.synchronize(dev)
        clk.wait_lines(1)
    if world > 1:
        dist.barrier()
    launches = launches_per_step * a.steps
    total_ms = t0.elapsed_time(t1)
    t = torch.tensor([total_ms, eager_ms, *phase.mean(0).tolist()], dtype=torch.float64,
                     device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, eager_ms, model_ms, enc_ms, frame_ms, dec_ms = t.tolist()
    # in-HBM packing of the ICH1 payload (not on the round-trip path: the
    # stream is packed when it leaves HBM) and the decode of the packed form
    pk = [ev() for _ in range(3)]
    reps = 5
    pk[0].record(stream)
    for _ in range(reps):
        codec.frame_range(n, 0, k_chunks, codec.payload.data_ptr())
    pk[1].record(stream)
    for _ in range(reps):
        codec.decode(d_out, n)
    pk[2].record(stream)
    torch.cuda.synchronize(dev)
    pack_ms, dec_packed_ms = pk[0].elapsed_time(pk[1]) / reps, pk[1].elapsed_time(pk[2]) / reps
    pk[0].record(stream)
    for _ in range(reps):
        codec.directory(n)
    pk[1].record(stream)
    torch.cuda.synchronize(dev)
    frame_ms = pk[0].elapsed_time(pk[1]) / reps  # alone; in the step it runs beside the decode
    ms_step = total_ms / a.steps
    gbs = lambda b, ms: b / (ms * 1e-3) / 1e9  # noqa: E731

    # compression ratio (framed ICH1 size) vs empirical entropy
    counts = codec.counts.cpu().numpy().astype(np.float64)
    H = entropy_bits(counts / counts.sum())
    table = codec.read_table()
    framed = 24 + 3 + 2 * table.alphabet_size + 4 * k_chunks + 4 * k_chunks * N + 2 * total_words
    single_hdr = 16 + 3 + 2 * table.alphabet_size + 4 * N
    bpb = 8 * framed / n

    # roofline for the dominant kernels: algorithmic bytes per launch
    dec_bytes = 2 * total_words + 4 * N * k_chunks + n          # payload + states read, raw written
    enc_bytes = n + 2 * total_words + 4 * N * k_chunks          # raw read, payload + states written
    hbm, peak_src = hbm_peak()
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():  # dram bytes per launch from the committed ncu --set full capture
        t = json.loads(tf.read_text())
        if t.get("config") == f"mib={n / MIB:g},chunk={C},lanes={N},sb={sb}":
            traffic = t
    dom = "decode" if dec_ms >= enc_ms else "encode"
    dom_ms = max(dec_ms, enc_ms)
    dom_bytes = dec_bytes if dom == "decode" else enc_bytes
    achieved = gbs(dom_bytes, dom_ms)

    out = {
        "metric": METRIC,
        "value": gbs(global_bytes, ms_step),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": a.steps,
        "warmup": a.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if a.global_mib else "weak",
        "vs_baseline": None,
        "dtype": "u8 symbols / u32 states / u16 digits (integer)",
        "data": "synthetic (counter-based splitmix64 Zipf sampler, csrc/synth.cu)",
        "config": config_of(a, world),
        "decode": {"GBps": gbs(n, dec_ms), "ms": dec_ms,
                   "roofline_frac": gbs(dec_bytes, dec_ms) / hbm},
        "encode": {"GBps": gbs(n, enc_ms), "ms": enc_ms, "kernel_ms": enc_ms,
                   "directory_ms": frame_ms,
                   "directory": "ICH1 word-offset scan, timed alone; in the step it runs on a "
                                "side stream beside the decode",
                   "roofline_frac": gbs(enc_bytes, enc_ms) / hbm},
        "pack": {"ms": pack_ms, "GBps": gbs(n, pack_ms),
                 "what": "ICH1 payload packed in HBM (offset scan + compaction); off the "
                         "round-trip path: the stream is packed when it leaves HBM",
                 "decode_packed_ms": dec_packed_ms},
        "model_build": {"ms": model_ms, "GBps": gbs(n, model_ms)},
        "ratio": {"bits_per_byte": bpb, "entropy_bpb": H, "vs_entropy": bpb / H,
                  # the quantized model's ideal code length for this message
                  # (sum over symbols of sb - log2 f_s, from the counts)
                  "model_ideal_bpb": float(
                      (counts[: table.alphabet_size] * (table.scale_bits - np.log2(
                          np.maximum(table.freq_u32, 1).astype(np.float64)))).sum() / n),
                  "single_stream_bits_per_byte": 8 * (single_hdr + 2 * total_words
                                                      - 4 * N * (k_chunks - 1)) / n,
                  "framed_bytes": framed, "payload_words": total_words},
        "roofline": {"bound": "hbm", "kernel": f"{dom}_warp_kernel", "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": ((traffic or {}).get("dram_bytes") or {}).get(dom),
                     "algorithmic_bytes": dom_bytes, "peak_source": peak_src},
        "gpu_launches": int(launches),
        "timing": (("CUDA graph of one step replayed K times" if world == 1 else
                    "CUDA graphs of the step around the eager NCCL all-reduce")
                   if graph is not None else "eager steps")
                  + f"; eager steps: {eager_ms / a.steps:.4f} ms/step",
        "clocks": clk.summary(),
    }
    # the bound that actually binds the coders: shared-memory wavefronts (the
    # random-address table lookups) -- ncu's per-launch wavefront count over
    # this run's kernel time, against one wavefront per SM per clock
    # and the instruction-issue bound (one warp instruction per SMSP-clock)
    wf = ((traffic or {}).get("smem_wavefronts") or {}).get(dom)
    wi = ((traffic or {}).get("warp_instructions") or {}).get(dom)
    sm_mhz = out["clocks"].get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clks = dom_ms * 1e-3 * sm_mhz * 1e6
    if wf:
        per_clk = wf / (sms * clks)
        out["roofline"]["smem"] = {"wavefronts_per_launch": wf, "achieved_per_sm_clk": per_clk,
                                   "peak_per_sm_clk": 1.0, "frac": per_clk,
                                   "source": "ncu l1tex__data_pipe_lsu_wavefronts_mem_shared.sum "
                                             "(profiles/ncu_traffic.json) / live kernel time"}
    if wi:
        per_clk = wi / (4 * sms * clks)
        out["roofline"]["issue"] = {"warp_instructions_per_launch": wi,
                                    "achieved_per_smsp_clk": per_clk, "peak_per_smsp_clk": 1.0,
                                    "frac": per_clk,
                                    "source": "ncu smsp__inst_executed.sum / live kernel time"}

    out["fused_consumer"] = fused_consumer(codec, d_out, n, dev)
    big = n > (2 << 30)  # config 3 sizes: free the step's buffers for the legs below
    if rank == 0 and world == 1 and a.scale_bits != 14 and not big:
        out["sb14"] = other_precision(a, dev, d_msg, n, 14)
    if big:
        del codec, d_out
        torch.cuda.empty_cache()

    if not a.no_e2e:
        out["e2e"] = e2e(a, n, k_chunks, C, N, sb, dev, d_msg, allreduce, world, global_bytes,
                         slots=2 if big else 3)
    if rank == 0 and world == 1 and not a.no_plugin:
        out["plugin_e2e"] = plugin_e2e(d_msg[:n].cpu().numpy(), table, C, N)
    if rank == 0 and world == 1:
        out["config1"] = config1(ref=False)

    if rank == 0 and world == 1 and not a.no_cpu:
        msg_h = d_msg[:n].cpu().numpy()
        out["cpu_baseline"] = cpu_reference(msg_h, sb, C, N)
        out["cpu_baseline"].pop("wall_s", None)

    if a.sweep and rank == 0:
        out["sweep"] = sweep(a, dev)
    if a.stress and rank == 0:
        out["stress"] = stress(a, dev)
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))


def other_precision(a, dev, d_msg, n, sb, steps=10):
    """The same device-resident step at another probability precision
    (sb = 14 is the reference's default, rans.py:131-133 / CLI
    --scale-bits 14): step, encode and decode times on the same input."""
    import torch

    from paper_1402_3392_b200.chunked import DeviceCodec, n_chunks_for

    codec = DeviceCodec(n, a.chunk, a.lanes, sb, dev)
    d_out = torch.empty(n, dtype=torch.uint8, device=dev)
    k = n_chunks_for(n, a.chunk)
    stream = torch.cuda.current_stream(dev)

    def step(m=None):
        if m: m[0].record(stream)
        codec.histogram(d_msg, n)
        codec.build_table_from_counts()
        if m: m[1].record(stream)
        codec.encode(d_msg, n, frame=False)
        if m: m[2].record(stream)
        codec.directory(n)
        if m: m[3].record(stream)
        codec.decode_slots(d_out, n)
        if m: m[4].record(stream)

    codec.reset_status()
    step()
    codec.check_status()
    torch.cuda.synchronize(dev)
    if not torch.equal(d_out, d_msg[:n]):
        raise SystemExit(f"sb={sb} round-trip mismatch")
    for _ in range(3):
        step()
    marks = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(steps)]
    for m in marks:
        step(m)
    torch.cuda.synchronize(dev)
    ph = np.array([[m[j].elapsed_time(m[j + 1]) for j in range(4)] for m in marks]).mean(0)
    ms = float(np.mean([m[0].elapsed_time(m[4]) for m in marks]))
    words = int(codec.offsets[k])
    hbm, _ = hbm_peak()
    dec_bytes = 2 * words + 4 * a.lanes * k + n
    enc_bytes = n + 2 * words + 4 * a.lanes * k
    flags = int(codec.table.view(torch.int32)[3].item())
    return {"scale_bits": sb, "ms_per_step_eager": ms, "GBps": n / (ms * 1e-3) / 1e9,
            "model_ms": ph[0], "encode_kernel_ms": ph[1], "decode_ms": ph[3],
            "decode_GBps": n / (ph[3] * 1e-3) / 1e9, "encode_GBps": n / (ph[1] * 1e-3) / 1e9,
            "decode_roofline_frac": dec_bytes / (ph[3] * 1e-3) / 1e9 / hbm,
            "encode_roofline_frac": enc_bytes / (ph[1] * 1e-3) / 1e9 / hbm,
            "decode_lut": "packed32" if flags & 1 else "packed64" if flags & 4 else "two-lookup",
            "encode_record": ("quad16" if flags & 16 else "fast12" if flags & 8 else "fast" if flags & 2
                              else "generic"),
            "payload_bits_per_byte": 16 * words / n}


def sweep(a, dev):
    """Config 4: entropy x precision sweep (decode / encode GB/s, ratio)."""
    import torch

    from paper_1402_3392_b200.chunked import DeviceCodec, n_chunks_for
    from paper_1402_3392_b200.synth import ZIPF_S_FOR_ENTROPY, synth_device

    n = min(a.mib, 256) * MIB
    rows = []
    for H, s in ZIPF_S_FOR_ENTROPY.items():
        d_msg = synth_device(n, s, a.seed, device=dev)
        d_out = torch.empty(n, dtype=torch.uint8, device=dev)
        for sb in range(11, 16):
            codec = DeviceCodec(n, a.chunk, a.lanes, sb, dev)
            codec.histogram(d_msg, n)
            codec.build_table_from_counts()
            codec.reset_status()
            codec.encode(d_msg, n)
            codec.decode(d_out, n)
            codec.check_status()
            assert torch.equal(d_out, d_msg[:n])
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            reps = 3
            ev[0].record()
            for _ in range(reps):
                codec.encode(d_msg, n)
            ev[1].record()
            for _ in range(reps):
                codec.decode(d_out, n)
            ev[2].record()
            torch.cuda.synchronize(dev)
            k = n_chunks_for(n, a.chunk)
            words = int(codec.offsets[k])
            rows.append({"H_target": H, "zipf_s": s, "scale_bits": sb,
                         "encode_GBps": n * reps / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9,
                         "decode_GBps": n * reps / (ev[1].elapsed_time(ev[2]) * 1e-3) / 1e9,
                         "payload_bits_per_byte": 16 * words / n})
    return rows


def stress(a, dev):
    """Config 5: small-chunk stress -- chunk sizes 64 KiB down to 4 KiB over
    the same 256 MiB (4 K .. 64 K streams) and 1 GiB of 64 KiB chunks (16 K
    streams, several waves): encode (kernel + framing) and decode GB/s, and
    the framing overhead (framed ICH1 bits/byte vs one stream's payload)."""
    import torch

    from paper_1402_3392_b200.chunked import DeviceCodec, n_chunks_for
    from paper_1402_3392_b200.synth import entropy_bits, synth_device

    rows = []
    for mib, C in ((256, 65536), (256, 16384), (256, 4096), (1024, 65536)):
        n = mib * MIB
        d_msg = synth_device(n, a.zipf_s, a.seed, device=dev)
        d_out = torch.empty(n, dtype=torch.uint8, device=dev)
        codec = DeviceCodec(n, C, a.lanes, a.scale_bits, dev)
        codec.histogram(d_msg, n)
        codec.build_table_from_counts()
        codec.reset_status()
        codec.encode(d_msg, n)
        codec.decode(d_out, n)
        codec.check_status()
        assert torch.equal(d_out, d_msg[:n])
        reps = 5
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        for _ in range(reps):
            codec.encode(d_msg, n)
        ev[1].record()
        for _ in range(reps):
            codec.decode(d_out, n)
        ev[2].record()
        torch.cuda.synchronize(dev)
        k = n_chunks_for(n, C)
        words = int(codec.offsets[k])
        alpha = codec.read_table().alphabet_size
        framed = 24 + 3 + 2 * alpha + 4 * k + 4 * k * a.lanes + 2 * words
        counts = codec.counts.cpu().numpy().astype(np.float64)
        rows.append({"bytes": n, "chunk_len": C, "streams": k,
                     "encode_GBps": n * reps / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9,
                     "decode_GBps": n * reps / (ev[1].elapsed_time(ev[2]) * 1e-3) / 1e9,
                     "framed_bits_per_byte": 8 * framed / n,
                     "entropy_bpb": entropy_bits(counts / counts.sum()),
                     "framing_overhead_bytes_per_chunk": (framed - 2 * words) / k})
        del codec, d_msg, d_out
        torch.cuda.empty_cache()
    return rows


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(max(1, a.gpus))))
    if rank != 0:
        return
    # the reference arm must not import this package (its __init__ loads
    # libilans_b200.so): the host sampler is loaded by file path
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "ilans_b200_synth_host", ROOT / "paper_1402_3392_b200" / "synth.py")
    synth = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(synth)
    synth_host = synth.synth_host

    n = a.global_mib * MIB // world if a.global_mib else a.mib * MIB
    cores = len(os.sched_getaffinity(0))
    per_core = 16  # MiB per core per step -> a bounded sample (16 cores: all 256 MiB)
    sample = min(n, cores * per_core * MIB)
    msg = synth_host(sample, a.zipf_s, a.seed)
    vals = []
    for i in range(a.warmup + a.steps):
        r = cpu_reference(msg, a.scale_bits, a.chunk, a.lanes, per_core_mib=per_core)
        if i >= a.warmup:
            vals.append(r)
    v = statistics.median([r["value"] for r in vals])
    ms = 1e3 * sample / (v * 1e9)
    base = vals[-1]
    base["value"] = v
    base.pop("wall_s", None)
    cfg1 = config1(ref=True)
    print(json.dumps({
        "config1": cfg1,
        "metric": METRIC, "impl": "reference", "value": v, "unit": "GB/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8 symbols / u32 states / u16 digits",
        "data": "synthetic (same sampler, host twin)", "config": config_of(a, world),
        "cpu_baseline": base,
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def launch_ranks(a) -> int:
    """``--gpus N`` (N > 1) outside torchrun: start N ranks, one per GPU,
    with torch.distributed.run on 127.0.0.1 (the driver's own launch form)
    and return their exit code. N larger than the visible GPUs is an error
    (``--dist-backend gloo`` may wrap ranks onto fewer GPUs for testing)."""
    import socket

    import torch

    visible = torch.cuda.device_count()
    if a.gpus > visible and a.dist_backend == "nccl":
        print(f"bench.py: --gpus {a.gpus} but only {visible} CUDA device(s) visible",
              file=sys.stderr)
        return 2
    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def run_plugin_only(a):
    from paper_1402_3392_b200.rans import SymbolTable
    from paper_1402_3392_b200.synth import synth_host

    msg = synth_host(256 * MIB, a.zipf_s, a.seed)
    counts = np.bincount(msg, minlength=256)
    table = SymbolTable.from_counts(counts[: int(np.nonzero(counts)[0][-1]) + 1].tolist(),
                                    a.scale_bits)
    print(json.dumps(plugin_e2e(msg, table, a.chunk, a.lanes,
                                threads_list=(1, 2, 4, 8, 16, 32))))


def main():
    a = parse()
    if a.plugin_only:
        run_plugin_only(a)
    elif a.impl == "reference":
        run_reference(a)
    elif a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(a))
    else:
        run_b200(a)
    # the line is printed: leave without the interpreter's teardown (one
    # --plugin-only run of many died with SIGSEGV after printing, during
    # CUDA / thread teardown at exit; the result is already out)
    sys.stdout.flush()
    sys.stderr.flush()
    os._exit(0)


if __name__ == "__main__":
    main()
