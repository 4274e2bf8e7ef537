#!/usr/bin/env python3
"""bench.py — Mpaths/s + Mlookups/s of the compressed-VDB path tracer (BASELINE.json metric).

Default workload (N=1, BASELINE configs[2] "C3"): 1024^3 ridged turbulence f32 -> 8-bit
fixed-rate VDB (AFFINE8 leaves, per-leaf lo/scale), 1920x1080 multi-bounce delta-tracking path
tracer (max_bounces 64, RR from bounce 3), 64 spp, seed 3. One step = one full frame.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3|C3_4bit|C5|C2|C1|C4]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)
  python bench.py --impl reference ...                 (the reference's CPU path, rank 0 only)

Multi-GPU: the volume is replicated, the image split into interleaved 16x16 tiles (tile t on
rank t % N), each rank renders its tiles into a packed device buffer, and one NCCL gather brings
them to rank 0 which un-interleaves them. Timing: CUDA events on the render stream, barrier +
synchronize around the K timed steps, max over ranks. ``value`` = all paths of all ranks / time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SECTOR_BYTES = 32  # algorithmic bytes per lookup (one HBM sector per random tap), SURVEY.md §8d
L2_BYTES = 126 << 20  # B200 L2
METRIC = "Mpaths/s (1024^3 8-bit compressed VDB path tracing; Mlookups/s alongside)"


def workload(sc):
    return (f"{sc.name}: {sc.dims[0]}x{sc.dims[1]}x{sc.dims[2]} {sc.volume} -> {sc.codec.name} leaves, "
            f"{sc.width}x{sc.height}, {sc.settings.spp} spp, {sc.settings.mode.name}, "
            f"max_bounces {sc.settings.max_bounces}")
L2_FLUSH_BYTES = 256 << 20  # written between timed steps when the leaf payload fits in L2


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
    ap.add_argument("--mode", default="", help="override the integrator: pathtrace|ratio|ea|iso")
    ap.add_argument("--precision", default="fp64", choices=["fp64", "fp32", "mixed"],
                    help="tracking arithmetic: fp64 reference-exact (bit parity), fp32 (tolerance parity)")
    ap.add_argument("--majorant-cell", type=int, default=0,
                    help="majorant grid edge: 0/32 reference macrocells (bit parity), 8 leaf, 128 lower node")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def scene_for(args):
    from dataclasses import replace
    from paper_2504_04564_b200 import scenes as S
    sc = S.scaled(args.config, args.scale, image_factor=1) if args.scale > 1 else S.SCENES[args.config]
    import paper_2504_04564_b200 as P
    st = replace(sc.settings, kernel=args.kernel, majorant_cell=args.majorant_cell,
                 precision={"fp64": 0, "fp32": 1, "mixed": 2}[args.precision])
    if args.spp:
        st = replace(st, spp=args.spp)
    if args.mode:
        st = replace(st, mode=P.RenderMode[args.mode])
    return replace(sc, width=args.width or sc.width, height=args.height or sc.height, settings=st)


def build_grid_bytes(sc, threads):
    import paper_2504_04564_b200 as P
    t0 = time.perf_counter()
    vol = P.synth(sc.volume, sc.dims, sc.volume_seed, threads=threads)
    t1 = time.perf_counter()
    svdb, rep = P.compress(vol, P.CompressionParams(1.0), voxel_type=sc.voxel_type, threads=threads)
    t2 = time.perf_counter()
    log(f"[bench] synth {sc.dims} {t1 - t0:.1f}s, compress {t2 - t1:.1f}s -> {len(svdb) / 1e9:.3f} GB SVDB")
    del vol
    return svdb, rep


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
def cpu_reference_sample(sc, svdb, codec, target_s, threads=0, tile_phase=0):
    """The reference CPU path (oracle/_ref, compiled from the unmodified sources) on a bounded
    tile sample of the same frame. Returns a dict with Mpaths/s and sample description."""
    from oracle.oracle import Oracle, Reference, have_reference
    if have_reference():
        kind = "reference"
        deq = svdb if codec == 0 else Oracle().quantize(svdb, codec)[0]
        rg = Reference().open(deq)
        cores = threads or Reference().hardware_threads()
        t0 = time.perf_counter()
        rg.macrocells(sc.tf)
        mc_s = time.perf_counter() - t0
        cam = sc.camera()
        tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
        stride = max(1, tiles // max(1, cores))  # ~1 tile per thread first
        rate = None
        while True:
            _, lk, pa, sec = rg.render_tiles(sc.tf, cam, sc.settings, tile_stride=stride, tile_phase=tile_phase % stride,
                                              threads=threads)
            rate = (pa / sec, lk / sec, pa, lk, sec, stride)
            if sec >= target_s * 0.5 or stride == 1:
                break
            grow = max(2.0, min(16.0, target_s / max(sec, 1e-3)))
            stride = max(1, int(stride / grow))
        pa_s, lk_s, pa, lk, sec, stride = rate
        return dict(value=pa_s / 1e6, unit="Mpaths/s", cores=cores, kind=kind,
                    mlookups_per_s=lk_s / 1e6, lookups_per_path=lk / max(pa, 1),
                    sample=(f"every {stride}th 16x16 tile of the {cam.width}x{cam.height} frame at full "
                            f"{sc.settings.spp} spp ({pa} paths, {sec:.1f} s, {cores} threads) on the "
                            f"dequantised grid; build_macrocells+update_majorants {mc_s:.1f} s "
                            "(not in the rate)"),
                    macrocell_seconds=mc_s)
    raise RuntimeError("oracle/_ref/libsvdbref.so missing: build it where /root/reference exists")


# ------------------------------------------------------------------------------------------
def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    sc = scene_for(args)
    import paper_2504_04564_b200 as P  # host encoder only (byte-identical to the reference's compress)
    svdb, _ = build_grid_bytes(sc, 0)
    codec = int(sc.codec)
    # size one step ~ a few seconds so warmup + steps stay within minutes
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    res = None
    times = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(sc, svdb, codec, per_step, tile_phase=i)
        if i >= args.warmup:
            times.append(r)
        res = r
    value = statistics.median([r["value"] for r in times]) if times else res["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value,
        "unit": "Mpaths/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(sc), "timed": "the unmodified reference's render_field body on "
                                                         "the host (oracle/_ref), bounded tile samples"},
        "mlookups_per_s": statistics.median([r["mlookups_per_s"] for r in times]) if times else None,
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": value, "unit": "Mpaths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2504_04564_b200 as P
    from paper_2504_04564_b200 import dist as D

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    sc = scene_for(args)
    cam = sc.camera()
    host_threads = max(1, (os.cpu_count() or 1) // max(1, world))
    svdb, rep = build_grid_bytes(sc, host_threads)
    t0 = time.perf_counter()
    grid = P.DeviceGrid(svdb, sc.codec, device=local)
    upload_s = time.perf_counter() - t0
    log(f"[bench] rank {rank}: grid on cuda:{local} codec {grid.codec.name}, device tree "
        f"{grid.device_bytes / 1e9:.3f} GB, upload+encode {upload_s:.1f}s")

    stream = torch.cuda.Stream(device=dev)
    flush_l2 = grid.leaf_payload_bytes < 2 * L2_BYTES
    ntiles = P.tiles_for_rank(cam.width, cam.height, rank, world)
    max_tiles = P.tiles_for_rank(cam.width, cam.height, 0, world)
    packed = torch.zeros(max_tiles * 768, dtype=torch.float32, device=dev)
    frame = torch.zeros(cam.height * cam.width * 3, dtype=torch.float32, device=dev) if rank == 0 else None

    def step():
        st = P.render_device(grid, sc.tf, cam, sc.settings, packed.data_ptr() if world > 1 else frame.data_ptr(),
                             stream.cuda_stream, packed=world > 1, tile_rank=rank, tile_nranks=world)
        if world > 1:
            with torch.cuda.stream(stream):
                allp = D.gather_packed(packed, world, rank)  # the only collective (NCCL)
                if rank == 0:
                    P.unpack_tiles_device(allp.data_ptr(), world, max_tiles, cam.width, cam.height,
                                          frame.data_ptr(), stream.cuda_stream)
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
    if world > 1:
        t = torch.tensor([ms, paths, lookups, samples, launches, sum(render_ms)], dtype=torch.float64, device=dev)
        mx = t.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = t.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, render_max = float(mx[0]), float(mx[5])
        paths, lookups, samples, launches = int(sm[1]), int(sm[2]), int(sm[3]), int(sm[4])
    else:
        render_max = sum(render_ms)

    # ---- the mixed-precision tracking variant of the same workload (precision=2: FP64 geometry,
    # FP32 step / sampler / TF arithmetic), timed the same way, and its distance to the FP64 frame
    # at matched streams (north-star tolerance: relative RMSE <= 1e-3) ----
    fp32 = None
    if world == 1 and not args.no_fp32 and sc.settings.precision == 0 and args.kernel == 0 and \
            sc.settings.mode in (P.RenderMode.pathtrace, P.RenderMode.ratio):
        from dataclasses import replace as _replace
        ref_frame = frame.clone()
        st32 = _replace(sc.settings, precision=2)
        P.render_device(grid, sc.tf, cam, st32, frame.data_ptr(), stream.cuda_stream)
        torch.cuda.synchronize(dev)
        d = (frame.double() - ref_frame.double())
        rel_rmse = float(torch.sqrt((d * d).sum() / (ref_frame.double() ** 2).sum().clamp_min(1e-300)))
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

    # ---- e2e through the C-ABI host-buffer call (svdbgpu_render): H2D of the TF, D2H image ----
    e2e = None
    if not args.no_e2e:
        rgb = np.zeros((cam.height, cam.width, 3), np.float32)
        import ctypes as C
        from paper_2504_04564_b200 import _native as N
        ctf, ccam, cst = sc.tf._c(), cam._c(), sc.settings._c(rank, world)
        st = N.Stats()
        L = N.lib()
        L.svdbgpu_render(grid.handle, C.byref(ctf), C.byref(ccam), C.byref(cst), rgb.ctypes.data, C.byref(st))
        if world > 1:
            dist.barrier()
        e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            rc = L.svdbgpu_render(grid.handle, C.byref(ctf), C.byref(ccam), C.byref(cst), rgb.ctypes.data,
                                  C.byref(st))
            if rc:
                raise RuntimeError(L.svdbgpu_last_error().decode())
        e_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([e_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_s = float(t[0])
        e_paths = cam.width * cam.height * sc.settings.spp * e_steps
        d2h = (ntiles * 256 if world > 1 else cam.width * cam.height) * 12
        e2e = {"value": e_paths / e_s / 1e6, "unit": "Mpaths/s", "steps": e_steps,
               "h2d_bytes_per_step": int(len(sc.tf.entries) * 16), "d2h_bytes_per_step": int(d2h),
               "note": "svdbgpu_render() host-buffer C-ABI call per frame: TF upload, majorants, render, "
                       "image D2H (wall clock, max over ranks)"}

    if rank == 0:
        peak, peak_src = peaks()
        s = ms / 1e3
        value = paths / s / 1e6
        # dominant kernel: k_render; achieved = algorithmic bytes per launch / avg launch time
        launch_s = render_max / 1e3 / args.steps
        per_launch_lookups = lookups / args.steps / world
        achieved = per_launch_lookups * SECTOR_BYTES / launch_s / 1e9
        traffic, prof = (ncu_traffic(args.config, paths / args.steps / world)
                         if args.scale == 1 and args.kernel == 0 and not args.mode
                         and args.majorant_cell in (0, 32) and args.precision == "fp64" else (None, None))
        line = {
            "metric": METRIC,
            "value": value, "unit": "Mpaths/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": ["f64", "f32", "f64/f32"][sc.settings.precision], "data": "synthetic",
            "config": {"workload": workload(sc),
                       "majorant_cell": sc.settings.majorant_cell or 32,
                       "image_split": f"interleaved 16x16 tiles over {world} GPU(s), NCCL gather to rank 0",
                       "l2": (f"L2 flushed between timed steps ({L2_FLUSH_BYTES >> 20} MB write outside the "
                              f"step events; leaf payload {grid.leaf_payload_bytes / 1e6:.1f} MB)" if flush_l2 else
                              "inputs larger than L2 (leaf payload "
                              f"{grid.leaf_payload_bytes / 1e9:.2f} GB vs 126 MB L2)"),
                       "device_tree_bytes": grid.device_bytes, "svdb_bytes": len(svdb)},
            "mlookups_per_s": lookups / s / 1e6,
            "samples_per_path": samples / max(paths, 1),
            "lookups_per_path": lookups / max(paths, 1),
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": prof.get("report") if prof else None,
                         "algorithmic_bytes_per_launch": per_launch_lookups * SECTOR_BYTES,
                         "kernel": "k_trace / k_render (CUDA events around the launch on its stream)",
                         "model": "32 B (one sector) per lattice lookup, 8 lookups per trilinear sample",
                         "peak_source": peak_src,
                         "note": ("leaf payload fits in L2: taps are served on chip after the first touch, so the "
                                  "32 B/lookup model overstates HBM bytes and frac can exceed 1" if flush_l2 else None)},
            "clocks": clk,
        }
        if e2e:
            line["e2e"] = e2e
        if fp32:
            line["mixed_precision_tracking"] = fp32
        if world == 1 and not args.no_cpu_baseline:
            try:
                cb = cpu_reference_sample(sc, svdb, int(grid.codec), args.cpu_seconds)
                line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
                line["cpu_baseline"]["mlookups_per_s"] = cb["mlookups_per_s"]
            except Exception as exc:  # reported, never fatal for the GPU number
                line["cpu_baseline"] = {"error": str(exc)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
