#!/usr/bin/env python3
"""bench.py — Mpaths/s + Mlookups/s of the compressed-VDB path tracer (BASELINE.json metric).

Default workload (N=1, BASELINE configs[2] "C3"): 1024^3 ridged turbulence f32 -> 8-bit
fixed-rate VDB (AFFINE8 leaves, per-leaf lo/scale), 1920x1080 multi-bounce delta-tracking path
tracer (max_bounces 64, RR from bounce 3), 64 spp, seed 3. One step = one full frame.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3|C3_4bit|C5|C2|C1|C4]
  python bench.py --gpus N ...          (no WORLD_SIZE: re-launches itself under torch.distributed.run)
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)
  python bench.py --impl reference ...  (the unmodified reference's CPU path, rank 0 only)
  python bench.py --mode sample         (K2: standalone sampler, Mlookups/s, random + ray-coherent)

Multi-GPU: the volume is replicated (rank 0 encodes it once and shares the SVDB bytes through
/dev/shm), the image is split into interleaved 16x16 tiles (tile t on rank t % N), each rank renders
its tiles into a packed device buffer, and one NCCL gather brings them to rank 0, which
un-interleaves them. Timing: CUDA events on the render stream, barrier + synchronize around the K
timed steps, max over ranks. ``value`` = all paths of all ranks / time.

The reference arm never loads the product library: its volume comes from the oracle's C restatement
of the synthetic generators (bit-identical, tests/test_synth.py) and its grid from the reference's
own compress().
"""
from __future__ import annotations

import argparse
import json
import mmap
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SECTOR_BYTES = 32  # algorithmic bytes per lookup (one HBM sector per random tap), SURVEY.md §8d
L2_BYTES = 126 << 20  # B200 L2
L2_FLUSH_BYTES = 256 << 20  # written between timed steps when the leaf payload fits in L2
METRIC = "Mpaths/s (1024^3 8-bit compressed VDB path tracing; Mlookups/s alongside)"
SAMPLE_METRIC = "Mlookups/s (K2 standalone trilinear sampler, 1024^3 8-bit compressed VDB)"


def workload(sc):
    return (f"{sc.name}: {sc.dims[0]}x{sc.dims[1]}x{sc.dims[2]} {sc.volume} -> {sc.codec.name} leaves, "
            f"{sc.width}x{sc.height}, {sc.settings.spp} spp, {sc.settings.mode.name}, "
            f"max_bounces {sc.settings.max_bounces}")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--scale", type=int, default=1, help="shrink the volume by this factor (profiling only)")
    ap.add_argument("--width", type=int, default=0)
    ap.add_argument("--height", type=int, default=0)
    ap.add_argument("--spp", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target CPU sample duration")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the mixed-precision side measurement")
    ap.add_argument("--kernel", type=int, default=0, help="0 auto (path-regenerating), 1 per-pixel (A/B)")
    ap.add_argument("--mode", default="",
                    help="override the integrator: pathtrace|ratio|ea|iso; 'sample' = K2 sampler benchmark")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32", "mixed"],
                    help="tracking arithmetic: fp64 reference-exact (bit parity), fp32 (tolerance parity)")
    ap.add_argument("--majorant-cell", type=int, default=0,
                    help="majorant grid edge: 0/32 reference macrocells (bit parity), 8 leaf, 128 lower node")
    ap.add_argument("--hdda", action="store_true", help="hierarchical empty-space skipping over the node tree")
    ap.add_argument("--lookups", type=int, default=1 << 26, help="K2: positions per sampler launch")
    ap.add_argument("--cpu-check", action="store_true",
                    help="launch-path check without GPUs: gloo ranks, encode-once sharing, per-rank tile render "
                         "(C oracle stand-in), the product gather + un-interleave, compared with a full frame")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def loaded_native():
    """Shared objects of this repo mapped into the process (what the driver records)."""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                p = line.split()[-1] if line.strip() else ""
                if p.endswith(".so") or ".so." in p:
                    if p.startswith(ROOT):
                        out.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(out)


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def scene_for(args):
    """The config as plain data (scenes.py is pure Python: importing it loads no native code)."""
    from dataclasses import replace
    from paper_2504_04564_b200 import scenes as S
    from paper_2504_04564_b200.api import RenderMode
    sc = S.scaled(args.config, args.scale, image_factor=1) if args.scale > 1 else S.SCENES[args.config]
    st = replace(sc.settings, kernel=args.kernel, majorant_cell=args.majorant_cell,
                 precision={"fp64": 0, "fp32": 1, "mixed": 2}[args.precision], hdda=int(args.hdda))
    if args.spp:
        st = replace(st, spp=args.spp)
    if args.mode and args.mode != "sample":
        st = replace(st, mode=RenderMode[args.mode])
    return replace(sc, width=args.width or sc.width, height=args.height or sc.height, settings=st)


def peak_rss_gb():
    import resource
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6  # ru_maxrss is in KB on Linux


def build_grid_bytes(sc, threads, device=0):
    """The grid's SVDB v1 bytes (byte-identical to the reference's compress + serialize_frozen). The
    fBm-based volumes go through the streaming device encoder (svdbgpu_synth_compress: no dense host
    array); Marschner-Lobb (host libm) through svdbgpu_synth + the native host encoder."""
    import paper_2504_04564_b200 as P
    if sc.volume != "marschner_lobb" and P.device_count() > device:
        svdb, rep, sec = P.synth_compress(sc.volume, sc.dims, sc.volume_seed, P.CompressionParams(1.0), device=device)
        info = {"encoder": "streaming device encoder (svdbgpu_synth_compress, 32-slice slabs)", "encode_s": sec,
                "peak_host_rss_gb": peak_rss_gb(), "n_leaf": int(np.frombuffer(svdb[52:60], np.uint64)[0])}
        log(f"[bench] streaming encode {sc.dims} {sec:.1f}s -> {len(svdb) / 1e9:.3f} GB SVDB, "
            f"peak host RSS {info['peak_host_rss_gb']:.1f} GB")
        return svdb, info
    t0 = time.perf_counter()
    vol = P.synth(sc.volume, sc.dims, sc.volume_seed, threads=threads)
    t1 = time.perf_counter()
    svdb, rep = P.compress(vol, P.CompressionParams(1.0), voxel_type=sc.voxel_type, threads=threads)
    t2 = time.perf_counter()
    log(f"[bench] synth {sc.dims} {t1 - t0:.1f}s, compress {t2 - t1:.1f}s -> {len(svdb) / 1e9:.3f} GB SVDB")
    del vol
    return svdb, {"encoder": "host (svdbgpu_synth + svdbgpu_compress)", "synth_s": t1 - t0, "compress_s": t2 - t1,
                  "peak_host_rss_gb": peak_rss_gb()}


def shared_grid_bytes(sc, rank, world, dist, threads, device=0):
    """Encode once: rank 0 builds the SVDB and publishes it in /dev/shm, the other ranks map it."""
    if world == 1:
        return build_grid_bytes(sc, threads, device)
    path = f"/dev/shm/svdb_bench_{os.environ.get('MASTER_PORT', '0')}_{sc.name}.svdb"
    info = {}
    if rank == 0:
        svdb, info = build_grid_bytes(sc, threads, device)
        tmp = path + ".tmp"
        with open(tmp, "wb") as f:
            f.write(svdb)
        os.replace(tmp, path)
        del svdb
    dist.barrier()
    with open(path, "rb") as f:
        mm = mmap.mmap(f.fileno(), 0, prot=mmap.PROT_READ)
    dist.barrier()
    if rank == 0:
        os.unlink(path)  # the mappings stay valid
    return mm, info


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.idx = device_index
        self.proc = None
        self.f = None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(5)
        except Exception:
            self.proc.kill()
        self.f.flush()
        self.f.seek(0)
        rows = [r.split(",") for r in self.f.read().strip().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for k, name in enumerate(names):
                    if r[5 + k].strip() == "Active":
                        reasons.add(name)
            except (ValueError, IndexError):
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config_key, paths_per_launch):
    """DRAM bytes per render launch: the committed `ncu --set full` capture's
    dram__bytes_read.sum + dram__bytes_write.sum per path (profiles/ncu_render_summary.json)
    times this launch's paths. None when no capture exists for the config."""
    p = os.path.join(ROOT, "profiles", "ncu_render_summary.json")
    try:
        with open(p) as f:
            e = json.load(f)[config_key]
        return e["dram_bytes_per_path"] * paths_per_launch, e
    except Exception:
        return None, None


# ------------------------------------------------------------------------------------------
# CPU side: the unmodified reference (oracle/_ref) and, for the new integrators, the C oracle
class CpuReference:
    """The reference's render body (render.hpp:295-310: Rng::for_pixel_sample, camera_ray,
    trace_path through the stock GridField) over the same grid, on the host cores."""

    def __init__(self, sc, svdb, codec):
        from oracle.oracle import Oracle, Reference, have_reference
        if not have_reference():
            raise RuntimeError("oracle/_ref/libsvdbref.so missing: build it where /root/reference exists")
        self.sc = sc
        self.cam = sc.camera()
        self.R = Reference()
        self.orc = Oracle()
        # quantised codecs: the image oracle is the reference on the dequantised grid
        self.svdb = svdb if codec == 0 else self.orc.quantize(bytes(svdb), codec)[0]
        self.rg = self.R.open(self.svdb)
        self.cores = self.R.hardware_threads()
        t0 = time.perf_counter()
        self.rg.macrocells(sc.tf)
        self.macrocell_s = time.perf_counter() - t0
        self.tiles = ((self.cam.width + 15) // 16) * ((self.cam.height + 15) // 16)

    def pass_(self, stride, phase, threads=0, count=False, rgb=None):
        rgb, lk, pa, sec = self.rg.render_tiles(self.sc.tf, self.cam, self.sc.settings, tile_stride=stride,
                                                tile_phase=phase % stride, threads=threads, rgb=rgb, count=count)
        return rgb, lk, pa, sec

    def spread(self, stride):
        """A stride coprime to the tile row length, so a subset samples every column of the frame."""
        import math
        tx = (self.cam.width + 15) // 16
        stride = max(1, min(stride, self.tiles))
        while stride > 1 and math.gcd(stride, tx) != 1:
            stride += 1
        return stride

    def stride_for(self, seconds, threads=0, start=64):
        """Tile stride whose pass takes about `seconds` (calibrated on a 1/start sample)."""
        st = self.spread(start)
        _, _, pa, sec = self.pass_(st, st - 1, threads=threads)
        rate = pa / max(sec, 1e-6)
        paths_frame = self.cam.width * self.cam.height * self.sc.settings.spp
        return self.spread(int(round(paths_frame / max(rate * seconds, 1.0))))

    def lookups_per_path(self):
        st = self.spread(max(1, self.tiles // 64))
        _, lk, pa, _ = self.pass_(st, 0, count=True)
        return lk / max(pa, 1)

    def describe(self, stride, n):
        return (f"{n} pass(es) over every {stride}th 16x16 tile of the {self.cam.width}x{self.cam.height} frame "
                f"(disjoint tile phases) at full {self.sc.settings.spp} spp, stock GridField, on the "
                f"{'dequantised ' if self.svdb is not None else ''}grid; build_macrocells+update_majorants "
                f"{self.macrocell_s:.1f} s (not in the rate)")


def cpu_baseline(sc, svdb, codec, target_s):
    """cpu_baseline for the GPU arm: best of 3 all-thread passes over disjoint tile phases (~target/3 s
    each), a 1-thread pass, lookups/path from an untimed counting pass. Returns (dict, reference image
    with the rendered tiles, mask of rendered pixels)."""
    ref = CpuReference(sc, svdb, codec)
    cam = ref.cam
    stride = ref.stride_for(target_s / 3.0)
    stride = max(stride, 3) if ref.tiles >= 3 else 1
    img = np.zeros((cam.height, cam.width, 3), np.float32)
    rates, paths, secs = [], 0, 0.0
    for ph in range(min(3, stride)):
        _, _, pa, sec = ref.pass_(stride, ph, rgb=img)
        rates.append(pa / sec / 1e6)
        paths += pa
        secs += sec
    st1 = ref.stride_for(3.0, threads=1, start=max(64, ref.tiles // 8))
    _, _, pa1, sec1 = ref.pass_(st1, 1, threads=1)
    lpp = ref.lookups_per_path()
    mask = np.zeros((cam.height, cam.width), bool)
    tx = (cam.width + 15) // 16
    for t in range(ref.tiles):
        if t % stride < min(3, stride):
            y0, x0 = (t // tx) * 16, (t % tx) * 16
            mask[y0:y0 + 16, x0:x0 + 16] = True
    best = max(rates)
    cb = {"value": best, "unit": "Mpaths/s", "cores": ref.cores, "kind": "reference",
          "cpu_model": cpu_model(), "best_of": len(rates), "rates": rates,
          "one_thread": {"value": pa1 / sec1 / 1e6, "unit": "Mpaths/s", "cores": 1,
                         "sample": f"every {st1}th tile, {pa1} paths, {sec1:.1f} s"},
          "mlookups_per_s": best * lpp, "lookups_per_path": lpp,
          "sample": ref.describe(stride, len(rates)) + f"; {paths} paths in {secs:.1f} s",
          "macrocell_seconds": ref.macrocell_s}
    return cb, img, mask, ref


def image_parity(got, want, mask):
    g = got[mask].astype(np.float64)
    w = want[mask].astype(np.float64)
    same = float(np.mean(np.all(got[mask].view(np.uint32) == want[mask].view(np.uint32), axis=-1)))
    d = g - w
    den = float(np.sqrt(np.mean(w * w))) or 1.0
    return {"identical_px": same, "rel_rmse": float(np.sqrt(np.mean(d * d))) / den,
            "max_abs": float(np.max(np.abs(d))) if d.size else 0.0, "pixels": int(mask.sum())}


# ------------------------------------------------------------------------------------------
def run_reference_arm(args):
    """--impl reference: the unmodified reference's CPU path on the same workload. No product code:
    volume from the oracle's restated synth, grid from the reference's compress()."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import Oracle, Reference
    sc = scene_for(args)
    t0 = time.perf_counter()
    vol = Oracle().synth(sc.volume, sc.dims, sc.volume_seed)
    t1 = time.perf_counter()
    svdb, _ = Reference().compress(vol, int(sc.voxel_type), 1.0, 2)
    t2 = time.perf_counter()
    del vol
    log(f"[reference] synth (oracle) {t1 - t0:.1f}s, reference compress {t2 - t1:.1f}s -> {len(svdb) / 1e9:.3f} GB")
    ref = CpuReference(sc, svdb, int(sc.codec))
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    stride = ref.stride_for(per_step)
    rates = []
    for i in range(args.warmup + args.steps):
        _, _, pa, sec = ref.pass_(stride, i)
        if i >= args.warmup:
            rates.append(pa / sec / 1e6)
    value = statistics.median(rates)
    lpp = ref.lookups_per_path()
    so = loaded_native()
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "Mpaths/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(sc),
                   "timed": "the unmodified reference's render_field body (oracle/_ref, stock GridField) on "
                            "the host, bounded tile samples; median over the timed steps",
                   "input": "volume: oracle/synth_oracle.c (bit-identical to the product synth); grid: the "
                            "reference's compress(); quantised codecs dequantised by the C oracle"},
        "mlookups_per_s": value * lpp, "lookups_per_path": lpp,
        "cpu_baseline": {"value": value, "unit": "Mpaths/s", "cores": ref.cores, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": ref.describe(stride, len(rates)),
                         "rates": rates},
        "e2e": {"value": value, "unit": "Mpaths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_so_loaded": so,
    }
    assert not any("libsvdbgpu" in p for p in so), "the reference arm must not load the product library"
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
def spawn_ranks(args):
    """--gpus N without a launcher: re-run this script under torch.distributed.run, one rank per GPU."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    log(f"[bench] launching {args.gpus} ranks: {' '.join(cmd)}")
    return subprocess.call(cmd)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2504_04564_b200 as P
    from paper_2504_04564_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    nccl = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        nccl = {"version": ".".join(str(v) for v in torch.cuda.nccl.version()),
                "comm_nranks": dist.get_world_size(), "backend": dist.get_backend()}
        log(f"[bench] rank {rank}: NCCL {nccl['version']} comm of {nccl['comm_nranks']} ranks")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    sc = scene_for(args)
    cam = sc.camera()
    host_threads = max(1, os.cpu_count() or 1)
    svdb, enc = shared_grid_bytes(sc, rank, world, dist, host_threads, local)
    t0 = time.perf_counter()
    grid = P.DeviceGrid(svdb, sc.codec, device=local)
    upload_s = time.perf_counter() - t0
    log(f"[bench] rank {rank}: grid on cuda:{local} codec {grid.codec.name}, device tree "
        f"{grid.device_bytes / 1e9:.3f} GB, upload+encode {upload_s:.1f}s")

    stream = torch.cuda.Stream(device=dev)
    flush_l2 = grid.leaf_payload_bytes < 2 * L2_BYTES
    ntiles = P.tiles_for_rank(cam.width, cam.height, rank, world)
    max_tiles = P.tiles_for_rank(cam.width, cam.height, 0, world)
    packed = torch.zeros(max(1, max_tiles) * 768, dtype=torch.float32, device=dev)
    frame = torch.zeros(cam.height * cam.width * 3, dtype=torch.float32, device=dev) if rank == 0 else None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    per_rank = {"render_ms": [], "gather_ms": []}

    def step(timed=False):
        if timed:
            ev[0].record(stream)
        st = P.render_device(grid, sc.tf, cam, sc.settings, packed.data_ptr() if world > 1 else frame.data_ptr(),
                             stream.cuda_stream, packed=world > 1, tile_rank=rank, tile_nranks=world)
        if timed:
            ev[1].record(stream)
        if world > 1:
            with torch.cuda.stream(stream):
                allp = D.gather_packed(packed, world, rank)  # the only collective (NCCL)
                if rank == 0:
                    P.unpack_tiles_device(allp.data_ptr(), world, max_tiles, cam.width, cam.height,
                                          frame.data_ptr(), stream.cuda_stream)
        if timed:
            ev[2].record(stream)
            ev[2].synchronize()
            per_rank["render_ms"].append(ev[0].elapsed_time(ev[1]))
            per_rank["gather_ms"].append(ev[1].elapsed_time(ev[2]))
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    if flush_l2:
        # leaf payload fits in L2: overwrite L2 between timed steps, outside each step's events
        flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
        stats, ms = [], 0.0
        for k in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(k))
            ev0.record(stream)
            stats.append(step())
            ev1.record(stream)
            ev1.synchronize()
            ms += ev0.elapsed_time(ev1)
    else:
        ev0.record(stream)
        stats = [step() for _ in range(args.steps)]
        ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    if not flush_l2:
        ms = ev0.elapsed_time(ev1)
    paths = sum(s["paths"] for s in stats)
    lookups = sum(s["lookups"] for s in stats)
    samples = sum(s["samples"] for s in stats)
    render_ms = [s["render_ms"] for s in stats]
    launches = sum(s["launches"] for s in stats) + (args.steps if (world > 1 and rank == 0) else 0)
    ranks_detail = None
    if world > 1:
        t = torch.tensor([ms, paths, lookups, samples, launches, sum(render_ms)], dtype=torch.float64, device=dev)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, render_max = float(mx[0]), float(mx[5])
        paths, lookups, samples, launches = int(sm[1]), int(sm[2]), int(sm[3]), int(sm[4])
        # per-rank render / gather time of one more (untimed-region) step each, for the balance report
        step(timed=True)
        mine = torch.tensor([per_rank["render_ms"][-1], per_rank["gather_ms"][-1], ntiles], dtype=torch.float64,
                            device=dev)
        alld = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(alld, mine)
        ranks_detail = [{"rank": r, "render_ms": float(a[0]), "gather_ms": float(a[1]), "tiles": int(a[2])}
                        for r, a in enumerate(alld)]
    else:
        render_max = sum(render_ms)
    fp64_frame = frame.cpu().numpy().reshape(cam.height, cam.width, 3).copy() if rank == 0 else None

    # ---- the mixed-precision tracking variant of the same workload (precision=2: FP64 geometry,
    # FP32 step / sampler / TF arithmetic), timed the same way (side number, not the headline) ----
    fp32, mixed_frame = None, None
    if world == 1 and not args.no_fp32 and sc.settings.precision == 0 and args.kernel == 0 and not args.hdda and \
            sc.settings.mode in (P.RenderMode.pathtrace, P.RenderMode.ratio):
        from dataclasses import replace as _replace
        st32 = _replace(sc.settings, precision=2)
        P.render_device(grid, sc.tf, cam, st32, frame.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize(dev)
        mixed_frame = frame.cpu().numpy().reshape(cam.height, cam.width, 3).copy()
        d = mixed_frame.astype(np.float64) - fp64_frame.astype(np.float64)
        rel_rmse = float(np.sqrt((d * d).sum() / max((fp64_frame.astype(np.float64) ** 2).sum(), 1e-300)))
        k32 = max(1, min(args.steps, 3))
        ms32 = 0.0
        n32 = l32 = 0
        for _ in range(k32):
            if flush_l2:
                with torch.cuda.stream(stream):
                    flush.fill_(0.0)
            ev0.record(stream)
            st = P.render_device(grid, sc.tf, cam, st32, frame.data_ptr(), stream.cuda_stream)
            ev1.record(stream)
            ev1.synchronize()
            ms32 += ev0.elapsed_time(ev1)
            n32 += st["paths"]
            l32 += st["lookups"]
        fp32 = {"value": n32 / (ms32 / 1e3) / 1e6, "unit": "Mpaths/s", "steps": k32,
                "mlookups_per_s": l32 / (ms32 / 1e3) / 1e6,
                "roofline_frac": l32 * SECTOR_BYTES / (ms32 / 1e3) / 1e9 / peaks()[0],
                "rel_rmse_vs_fp64": rel_rmse, "dtype": "f64/f32",
                "note": "same workload with SVDBGPU_PRECISION_MIXED (FP64 ray/DDA/distances, FP32 step log, "
                        "sampler weights, TF, throughput); image compared with the FP64 frame above at "
                        "matched streams (north-star tolerance 1e-3)"}

    # ---- e2e through the public API with host buffers (svdbgpu_render: TF H2D, majorants, render,
    # image D2H), every timed step ----
    e2e = None
    if not args.no_e2e:
        # the result lands in pinned host memory (the copy runs at full PCIe speed)
        host_img = torch.empty((cam.height, cam.width, 3), dtype=torch.float32, pin_memory=True).numpy()
        P.render(grid, sc.tf, cam, sc.settings, tile_rank=rank, tile_nranks=world, out=host_img)
        if world > 1:
            dist.barrier()
        e_steps = max(1, args.steps)
        t0 = time.perf_counter()
        for _ in range(e_steps):
            P.render(grid, sc.tf, cam, sc.settings, tile_rank=rank, tile_nranks=world, out=host_img)
        e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_s = float(t[0])
        e_paths = cam.width * cam.height * sc.settings.spp * e_steps
        d2h = (ntiles * 256 if world > 1 else cam.width * cam.height) * 12
        e2e = {"value": e_paths / e_s / 1e6, "unit": "Mpaths/s", "steps": e_steps,
               "h2d_bytes_per_step": int(len(sc.tf.entries) * 16), "d2h_bytes_per_step": int(d2h),
               "note": "paper_2504_04564_b200.render() -> svdbgpu_render(): host TF upload, majorants, render, "
                       "image D2H into a pinned host buffer, per frame (wall clock, max over ranks)"}

    if rank == 0:
        peak, peak_src = peaks()
        s = ms / 1e3
        value = paths / s / 1e6
        # dominant kernel: k_trace; achieved = algorithmic bytes per launch / avg launch time
        launch_s = render_max / 1e3 / args.steps
        per_launch_lookups = lookups / args.steps / world
        achieved = per_launch_lookups * SECTOR_BYTES / launch_s / 1e9
        traffic, prof = (ncu_traffic(args.config, paths / args.steps / world)
                         if args.scale == 1 and args.kernel == 0 and not args.mode and not args.hdda
                         and args.majorant_cell in (0, 32) and args.precision == "fp64" else (None, None))
        line = {
            "metric": METRIC,
            "value": value, "unit": "Mpaths/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": ["f64", "f32", "f64/f32"][sc.settings.precision], "data": "synthetic",
            "config": {"workload": workload(sc),
                       "majorant_cell": sc.settings.majorant_cell or 32, "hdda": bool(args.hdda),
                       "image_split": f"interleaved 16x16 tiles over {world} GPU(s), NCCL gather to rank 0",
                       "l2": (f"L2 flushed between timed steps ({L2_FLUSH_BYTES >> 20} MB write outside the "
                              f"step events; leaf payload {grid.leaf_payload_bytes / 1e6:.1f} MB)" if flush_l2 else
                              "inputs larger than L2 (leaf payload "
                              f"{grid.leaf_payload_bytes / 1e9:.2f} GB vs 126 MB L2)"),
                       "device_tree_bytes": grid.device_bytes, "svdb_bytes": len(svdb),
                       "encode": enc, "upload_s": upload_s},
            "mlookups_per_s": lookups / s / 1e6,
            "samples_per_path": samples / max(paths, 1),
            "lookups_per_path": lookups / max(paths, 1),
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": prof.get("report") if prof else None,
                         "algorithmic_bytes_per_launch": per_launch_lookups * SECTOR_BYTES,
                         "kernel": "k_trace (CUDA events around the launch on its stream)",
                         "model": "32 B (one sector) per lattice lookup, 8 lookups per trilinear sample",
                         "peak_source": peak_src,
                         "note": ("leaf payload fits in L2: taps are served on chip after the first touch, so the "
                                  "32 B/lookup model overstates HBM bytes and frac can exceed 1" if flush_l2 else None)},
            "clocks": clk,
        }
        if nccl:
            line["nccl"] = nccl
        if ranks_detail:
            line["ranks"] = ranks_detail
        if e2e:
            line["e2e"] = e2e
        if fp32:
            line["mixed_precision_tracking"] = fp32
        if world == 1 and not args.no_cpu_baseline:
            try:
                cb, ref_img, mask, ref = cpu_baseline(sc, svdb, int(grid.codec), args.cpu_seconds)
                line["cpu_baseline"] = cb
                if sc.settings.mode == P.RenderMode.pathtrace and not args.hdda and \
                        sc.settings.majorant_cell in (0, 32):
                    par = image_parity(fp64_frame, ref_img, mask)
                    par["oracle"] = ("oracle/_ref: the unmodified reference's render body on the "
                                     f"{'dequantised ' if int(grid.codec) else ''}grid, same tiles")
                else:  # the new integrators / majorant grids: the C oracle (parity unpinned by reference)
                    from oracle.oracle import Oracle
                    stride = max(3, ref.tiles // 64)
                    oimg, _, _ = Oracle().open(ref.svdb).render(sc.tf, cam, sc.settings, tile_rank=0,
                                                                tile_nranks=stride)
                    m = np.zeros_like(mask)
                    tx = (cam.width + 15) // 16
                    for t in range(0, ref.tiles, stride):
                        m[(t // tx) * 16:(t // tx) * 16 + 16, (t % tx) * 16:(t % tx) * 16 + 16] = True
                    par = image_parity(fp64_frame, oimg, m)
                    par["oracle"] = f"oracle/svdb_oracle.c restatement, every {stride}th tile"
                par["tiles_fraction"] = float(mask.mean()) if "restatement" not in par["oracle"] else None
                if mixed_frame is not None and "restatement" not in par["oracle"]:
                    par["mixed"] = image_parity(mixed_frame, ref_img, mask)
                par["tolerance"] = "rel RMSE <= 1e-3 (north star)"
                line["parity"] = par
            except Exception as exc:  # reported, never fatal for the GPU number
                line["cpu_baseline"] = {"error": str(exc)}
        line["native_so_loaded"] = loaded_native()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------------------------
def run_sampler(args):
    """K2: standalone trilinear sampler (sample.hpp:46-72) at 1024^3 8-bit, random and
    ray-coherent position streams resident in HBM; Mlookups/s = 8 x samples/s; roofline on 32 B per
    lookup. One step = one launch over --lookups positions of each stream."""
    import torch

    import paper_2504_04564_b200 as P
    sc = scene_for(args)
    svdb, enc = build_grid_bytes(sc, max(1, os.cpu_count() or 1))
    grid = P.DeviceGrid(svdb, sc.codec, device=0)
    n = args.lookups
    gen = torch.Generator(device="cuda").manual_seed(7)
    hi = torch.tensor([d - 1 for d in sc.dims], dtype=torch.float64, device="cuda")
    streams = {"random": torch.rand((n, 3), dtype=torch.float64, device="cuda", generator=gen) * hi}
    # ray-coherent: 32 consecutive positions step 0.5 voxel along one random ray (a warp marches a ray)
    nr = n // 32
    o = torch.rand((nr, 1, 3), dtype=torch.float64, device="cuda", generator=gen) * hi
    d = torch.nn.functional.normalize(torch.randn((nr, 1, 3), dtype=torch.float64, device="cuda", generator=gen),
                                      dim=-1)
    k = torch.arange(32, dtype=torch.float64, device="cuda").view(1, 32, 1)
    streams["ray_coherent"] = torch.minimum(torch.maximum(o + d * k * 0.5, torch.zeros_like(hi)), hi).reshape(-1, 3)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    stream = torch.cuda.Stream()
    peak, peak_src = peaks()
    res = {}
    for name, xyz in streams.items():
        xyz = xyz.contiguous()
        m = xyz.shape[0]
        for _ in range(args.warmup):
            P.sample_device(grid, xyz.data_ptr(), m, 1, out.data_ptr(), stream.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            P.sample_device(grid, xyz.data_ptr(), m, 1, out.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 1e3
        mlk = 8 * m * args.steps / s / 1e6
        # position stream read (24 B) + output write (4 B) per sample are real HBM bytes too
        io = (24 + 4) * m * args.steps / s / 1e9
        res[name] = {"mlookups_per_s": mlk, "msamples_per_s": mlk / 8, "ms_per_launch": s * 1e3 / args.steps,
                     "roofline_frac": mlk * 1e6 * SECTOR_BYTES / 1e9 / peak, "stream_io_gbs": io}
    # parity spot check of the benchmarked kernel against the C oracle on the dequantised grid
    from oracle.oracle import Oracle
    xs = streams["random"][:4096].cpu().numpy()
    got = grid.sample(xs, 1)
    want = None
    try:
        deq = Oracle().quantize(bytes(svdb), int(grid.codec))[0] if int(grid.codec) else bytes(svdb)
        want = Oracle().open(deq).sample(xs, 1)
    except Exception as exc:  # noqa: BLE001
        log(f"[bench] sampler oracle check skipped: {exc}")
    line = {"metric": SAMPLE_METRIC, "value": res["random"]["mlookups_per_s"], "unit": "Mlookups/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"K2 sampler: {sc.name} grid {sc.dims[0]}^3 {sc.codec.name}, {n} positions per "
                                   "launch (random uniform in the box; ray-coherent: 32 steps of 0.5 voxel per ray)",
                       "l2": "inputs larger than L2"},
            "streams": res,
            "roofline": {"bound": "hbm", "achieved": res["random"]["mlookups_per_s"] * 1e6 * SECTOR_BYTES / 1e9,
                         "peak": peak, "unit": "GB/s", "frac": res["random"]["roofline_frac"], "traffic": None,
                         "peak_source": peak_src, "kernel": "k_sample"},
            "parity": ({"bit_exact": bool(np.array_equal(np.asarray(got).view(np.uint32),
                                                          np.asarray(want).view(np.uint32))), "n": len(xs)}
                       if got is not None and want is not None else None),
            "native_so_loaded": loaded_native()}
    print(json.dumps(line), flush=True)
    return 0


def run_cpu_check(args):
    """--cpu-check: the multi-rank plumbing of run_ours on CPU (gloo): spawn, encode once through
    /dev/shm, each rank renders its interleaved tiles (the C oracle stands in for k_trace), packs them,
    the product's gather_packed brings them to rank 0, which un-interleaves and compares the frame
    with a single-process render."""
    import torch
    import torch.distributed as dist

    from oracle.oracle import Oracle
    from paper_2504_04564_b200 import dist as D
    from paper_2504_04564_b200 import scenes as S
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    sc = S.scaled("C2", 8, spp=2, image_factor=10)
    cam = sc.camera()
    svdb, _ = shared_grid_bytes(sc, rank, world, dist, 2)
    img, _, _ = Oracle().open(bytes(svdb)).render(sc.tf, cam, sc.settings, tile_rank=rank, tile_nranks=world,
                                                  threads=2)
    n_max = D.max_tiles(cam.width, cam.height, world)
    packed = torch.from_numpy(D.pack_tiles(img, rank, world, pad_to=n_max))
    allp = D.gather_packed(packed, world, rank)
    if rank == 0:
        frame = D.unpack_tiles(allp.numpy(), world, n_max, cam.width, cam.height)
        full, _, _ = Oracle().open(bytes(svdb)).render(sc.tf, cam, sc.settings)
        print(json.dumps({"cpu_check": True, "n_gpus": args.gpus, "world": world,
                          "backend": dist.get_backend() if world > 1 else None,
                          "bit_identical": bool(np.array_equal(frame.view(np.uint32), full.view(np.uint32)))}),
              flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        return spawn_ranks(args)
    if env_world is not None and int(env_world) != args.gpus:
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE={env_world}: launch one rank per GPU "
            f"(torchrun --nproc-per-node {args.gpus}) or drop the launcher and let bench.py spawn them")
        return 2
    if args.cpu_check:
        return run_cpu_check(args)
    if args.mode == "sample":
        return run_sampler(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
