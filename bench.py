"""bench.py -- LucidRaster frame benchmark on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload stack64k|boxes1080|tiny4m|mixed16m]

A "step" is one frame of the workload through the full sort-middle pipeline
(setup -> binning -> low/high bin rasterization -> framebuffer). The default
workload is BASELINE.json configs[1] ("stack64k": 65,536 overlapping
translucent quads at 1920x1080, depth complexity ~32). N > 1 (torchrun, one
rank per GPU over NCCL) splits the frame's bins across ranks
(owner = (bx + 3*by) mod N, setup replicated) and gathers the finished 32x32
tiles to rank 0 over NVLink with NCCL; the frame time is the max over ranks.

value      = fragments per second of whole frames, all ranks (Gfragments/s)
ms_per_step = ms per frame (device time, CUDA events on the renderer's stream)
e2e        = the same metric through the reference-facing C ABI
             (veil_scene_set_camera + veil_render_scene + pixel readback into
             host memory) -- the headline number against the reference arm
roofline   = the dominant kernel (bin rasterizer) vs measured HBM bandwidth
cpu_baseline = the unmodified reference (oracle/_ref) on this host's cores
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ms/frame & Gfragments/s at 1920x1080 vs HBM roofline; at 1/2/4/8 B200"
L2_BYTES = 126 * 1024 * 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="stack64k",
                    choices=["stack64k", "boxes1080", "tiny4m", "mixed16m"])
    ap.add_argument("--df", type=int, default=3,
                    help="depth_filter_size (reference default 3; >8 runs the ring filter in memory)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="bound on the CPU-baseline sample (rank 0, N=1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo gathers tiles through host memory (orchestration tests)")
    ap.add_argument("--single-device", action="store_true",
                    help="every rank on cuda:0 (orchestration tests with --dist-backend gloo; "
                         "ranks never wait on each other inside kernels)")
    ap.add_argument("--gather", default="peer", choices=["peer", "nccl"],
                    help="N>1: sharded ranks write into rank 0's framebuffer over NVLink (CUDA IPC, "
                         "'peer') or pack tiles for an NCCL gather ('nccl')")
    ap.add_argument("--check-frame", action="store_true",
                    help="rank 0 compares the gathered frame with an unsharded render")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------- workloads

def orbit_eye(frame):
    """SURVEY.md 8(d) C3 camera path: 64 frames around the boxes."""
    import numpy as np

    R = float(np.hypot(5.5, 9.0))
    th = float(np.arctan2(5.5, 9.0)) + 2.0 * np.pi * (frame % 64) / 64.0
    return [R * np.sin(th), 4.5, R * np.cos(th)]


# Every workload's description; identical in both arms' `config`.
L2_NOTE = ("GPU arm: L2 flushed between timed frames (256 MiB write, outside the events); "
           "CPU reference arm: not applicable")
WORKLOADS = {
    "stack64k": {"workload": "stack64k", "quads": 65536, "width": 1920, "height": 1080, "seed": 2,
                 "depth_complexity": "~32", "baseline_config": 1},
    "boxes1080": {"workload": "boxes1080", "quads": 54, "width": 1920, "height": 1080,
                  "camera_path": "64-frame orbit", "baseline_config": 2},
    "tiny4m": {"workload": "tiny4m", "quads": 4194304, "width": 3840, "height": 2160, "seed": 4,
               "baseline_config": 3},
    "mixed16m": {"workload": "mixed16m", "quads": 16777216, "width": 7680, "height": 4320, "seed": 5,
                 "baseline_config": 4},
}


def workload_config(workload, df=3):
    return dict(WORKLOADS[workload], depth_filter_size=df, l2=L2_NOTE)


def workload_arrays(workload):
    """The workload's host arrays WITHOUT libveil (numpy restatement of the
    generators, oracle/workloads.py, checked equal to libveil's in
    tests/test_workloads_cpu.py; the boxes scene from its golden fixture)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    if workload == "boxes1080":
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from common import boxes_arrays

        return boxes_arrays(1920, 1080)
    import workloads

    return workloads.workload(workload, WORKLOADS[workload]["seed"])


def make_scene(workload, df=3):
    """Our arm: (veil.Scene, config, camera_fn or None); camera_fn(i) ->
    (matrix, eye) through libveil's look_at."""
    from paper_2405_13364_b200 import veil

    cfg = workload_config(workload, df)
    if workload == "boxes1080":
        s = veil.Scene.from_arrays(workload_arrays(workload))

        def cam(i):
            eye = orbit_eye(i)
            return veil.look_at(eye, [0, 0, 0], [0, 1, 0], 55.0, 0.5, 40.0, 1920, 1080), eye

        return s, cfg, cam
    return veil.Scene.workload(workload, cfg["seed"]), cfg, None


def reference_camera_fn(workload, lifted=False):
    """The same orbit through the reference's own make_look_at_camera
    (ref_shim vref_look_at; equal to libveil's, tests/test_workloads_cpu.py)."""
    if workload != "boxes1080":
        return None
    import bindings

    def cam(i):
        eye = orbit_eye(i)
        return bindings.ref_look_at(eye, [0, 0, 0], [0, 1, 0], 55.0, 0.5, 40.0, 1920, 1080, lifted), eye

    return cam


def reference_variant(arrays):
    """Which reference build can render this viewport: the unmodified one
    (<= 2560x2048), the limits-lifted one (<= 4096x4096, oracle/Makefile
    ref-lifted), or none."""
    if arrays.width <= 2560 and arrays.height <= 2048:
        return False
    if arrays.width <= 4096 and arrays.height <= 4096:
        return True
    return None


def bytes_model(stats, width, height, a_q=32, a_v=8):
    """SURVEY.md 8(d) algorithmic bytes (per frame, and the raster kernel's)."""
    Q, V = stats["input_quads"], stats["vertices"]
    Qv, Tv = stats["visible_quads"], 2 * stats["visible_quads"]
    Qs, Tl = stats["small_quads"], stats["large_tris"]
    P = stats["bin_pairs"]
    # split pairs into small-quad pairs and large-triangle pairs
    Ps, Pl = stats["pairs_small"], stats["pairs_large"]
    frame = (20 * Q + 12 * V + a_v * V + (4 + a_q) * Qv + 84 * Tv + 8 * Qs + 64 * Tl + 8 * P
             + (168 + a_q) * Ps + (84 + a_q) * Pl + 4 * width * height)
    raster = (168 + a_q) * Ps + (84 + a_q) * Pl + 4 * P + 5 * width * height
    b_min = 20 * Q + 12 * V + a_v * V + 8 * P + 4 * width * height
    return frame, raster, b_min


def ncu_summary(workload):
    """The committed ncu --set full capture of one frame's bin-rasterizer
    kernels (profiles/traffic.json, written by tools/ncu_traffic.py): DRAM
    bytes (read + write) per frame and the dominant kernel's issue-slot
    utilisation; empty when no capture exists."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload, {})
    except (OSError, ValueError):
        return {}


# ------------------------------------------------------------------- clocks

class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ------------------------------------------------------------- CPU baseline

def cpu_reference_run(arrays, frames_max, seconds, threads, camera_fn=None, lifted=False,
                      keep_first=False, depth_filter=3):
    """The unmodified reference (oracle/_ref; the limits-lifted build for
    viewports over 2560x2048) through its own C API, veil_render_scene.
    keep_first: also return the first frame's image and mask (camera 0)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bindings  # test/baseline infrastructure only
    from paper_2405_13364_b200.abi import default_params

    if lifted is None or not bindings.ref_available(lifted):
        return None
    rs = bindings.RefScene.from_arrays(arrays, lifted)
    p = default_params(thread_count=threads, depth_filter_size=depth_filter)
    times, frags = [], []
    first = None
    t_end = time.perf_counter() + seconds
    i = 0
    while i < frames_max and (i == 0 or time.perf_counter() < t_end):
        if camera_fn:
            m, eye = camera_fn(i)
            rs.set_camera(m, eye)
        t0 = time.perf_counter()
        img, mask, rep = rs.render(p)
        times.append(time.perf_counter() - t0)
        frags.append(rep["fragments"])
        if keep_first and first is None:
            first = (img, mask, rep)
        i += 1
    out = {"frames": len(times), "seconds": sum(times), "fragments": sum(frags),
           "gfrag_s": sum(frags) / sum(times) / 1e9, "ms_per_frame": 1e3 * sum(times) / len(times),
           "build": "lifted" if lifted else "unmodified"}
    if keep_first:
        out["first"] = first
    return out


def image_parity(got_img, got_mask, ref_img, ref_mask, against):
    """RGBA8 / invalid-mask comparison of one frame (north_star: <= 1/255 per
    channel, max-abs and PSNR stated)."""
    import numpy as np

    a = np.asarray(got_img, dtype=np.int16).reshape(-1, 4)
    b = np.asarray(ref_img, dtype=np.int16).reshape(-1, 4)
    d = np.abs(a - b)
    mse = float((d.astype(np.float64) ** 2).mean())
    return {"identical": bool(np.array_equal(a, b) and np.array_equal(got_mask, ref_mask)),
            "max_abs": int(d.max()) if d.size else 0,
            "psnr": None if mse == 0 else 10.0 * float(np.log10(255.0 ** 2 / mse)),
            "differing_px": int((d.max(axis=1) > 0).sum()),
            "mask_differing_px": int((np.asarray(got_mask).reshape(-1) != np.asarray(ref_mask).reshape(-1)).sum()),
            "against": against}


# ------------------------------------------------------------------ our arm

def device_bytes(ptr, n):
    """A torch uint8 view of n bytes of libveil device memory."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False),
                                    "version": 3, "strides": None}

    return torch.as_tensor(_View(), device="cuda")


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2405_13364_b200 import veil
    from paper_2405_13364_b200.abi import default_params

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.single_device:
        local = 0
    gloo = args.dist_backend == "gloo"
    cdev = "cpu" if gloo else "cuda"  # where collective tensors live
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # NCCL's init log (stderr) shows the communicator's ranks and transports
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    veil.set_device(local)

    scene, cfg, camera_fn = make_scene(args.workload, args.df)
    arrays = scene.arrays() if rank == 0 else None
    W, H = cfg["width"], cfg["height"]
    params = default_params(depth_filter_size=args.df)
    shard = (rank, world)
    stream = torch.cuda.ExternalStream(scene.stream())
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")
    bx, by = (W + 31) // 32, (H + 31) // 32
    counts = [veil.shard_tile_count(bx, by, r, world) for r in range(world)]
    max_tiles = max(counts)
    tiles = torch.empty(max_tiles * 5120, dtype=torch.uint8, device="cuda")
    gathered = ([torch.empty_like(tiles, device=cdev) for _ in range(world)]
                if (world > 1 and rank == 0) else None)

    peer = False
    if world > 1 and args.gather == "peer":
        # rank 0's framebuffer as CUDA IPC handles; the other ranks' shading
        # kernels then write their finished pixels straight into it
        blob = [veil.export_framebuffer(scene) if rank == 0 else None]
        dist.broadcast_object_list(blob, src=0)
        try:
            if rank != 0:
                veil.import_peer_framebuffer(scene, blob[0])
            ok = 1
        except veil.VeilError:
            ok = 0
        okt = torch.tensor([ok], dtype=torch.int32, device=cdev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        peer = bool(okt.item())
        if not peer and rank != 0:
            veil.import_peer_framebuffer(scene, None)

    def frame(i, timed_events=None):
        if camera_fn:
            m, eye = camera_fn(i)
            scene.set_camera(m, eye)
        if timed_events:
            # libveil records the start event right before the frame's graph
            # launch and (one GPU) the end event right after it, on the same
            # stream: the region is the frame's device work, without the
            # host's launch preparation or its wake-up after the frame's wait
            hs = timed_events[0].cuda_event
            he = timed_events[1].cuda_event if world == 1 else None
            veil.render_device(scene, params, shard, stats=False, events=(hs, he))
            if world == 1:
                return scene.last_stats()
        else:
            veil.render_device(scene, params, shard, stats=False)
        if peer:
            # every rank's pixels are in rank 0's framebuffer once all ranks'
            # frames completed (render_device synchronises its stream)
            if timed_events:
                timed_events[1].record(stream)
            dist.barrier()
            return scene.last_stats()
        if world > 1:
            veil.pack_tiles_device(scene, rank, world, tiles.data_ptr(), tiles.numel())
            with torch.cuda.stream(stream):
                mine = tiles.cpu() if gloo else tiles
                if rank == 0:
                    dist.gather(mine, gathered, dst=0)
                    for r in range(1, world):
                        g = gathered[r].to("cuda", non_blocking=False) if gloo else gathered[r]
                        veil.unpack_tiles_device(scene, r, world, g.data_ptr(), g.numel())
                        if gloo:
                            stream.synchronize()  # g is freed on return
                else:
                    dist.gather(mine, None, dst=0)
        if timed_events:
            timed_events[1].record(stream)
        return scene.last_stats()

    for i in range(args.warmup):
        frame(i)
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for a, b in evs:  # torch creates its events at their first record
        a.record(stream)
        b.record(stream)
    stats = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()  # L2 flush between timed frames (outside the events)
            stats.append(frame(args.warmup + i, evs[i]))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    ms_sum = torch.tensor([sum(ms)], dtype=torch.float64, device=cdev)
    frag_local = torch.tensor([sum(int(s.fragments) for s in stats)], dtype=torch.float64,
                              device=cdev)
    if world > 1:
        dist.all_reduce(ms_sum, op=dist.ReduceOp.MAX)
        dist.all_reduce(frag_local, op=dist.ReduceOp.SUM)
    ms_per_frame = float(ms_sum.item()) / args.steps
    fragments_per_frame = float(frag_local.item()) / args.steps
    value = fragments_per_frame / (ms_per_frame * 1e-3) / 1e9

    # --- e2e through the C ABI with host buffers (rank 0 owns the output)
    e2e = None
    if not args.no_e2e:
        if world == 1:
            e2e_ms = []
            for i in range(max(3, args.steps // 2)):
                if camera_fn:
                    m, eye = camera_fn(i)
                t0 = time.perf_counter()
                if camera_fn:
                    scene.set_camera(m, eye)
                r = veil.render(scene, params)
                px = r.pixels(copy=False)  # the handle's host RGBA8, as a C caller sees it
                mk = r.invalid_mask(copy=False)
                _ = int(px[-1, -1, 3]) + int(mk[-1, -1])  # touch the host data
                e2e_ms.append((time.perf_counter() - t0) * 1e3)
                del r
            e2e_ms = statistics.median(e2e_ms)
            e2e = {"value": fragments_per_frame / (e2e_ms * 1e-3) / 1e9, "unit": "Gfragments/s",
                   "ms_per_step": e2e_ms, "h2d_bytes_per_step": (128 + 64) if camera_fn else 64,
                   "d2h_bytes_per_step": int(px.nbytes + mk.nbytes),
                   "path": ("veil_scene_set_camera + " if camera_fn else "")
                           + "veil_render_scene + veil_render_pixels/veil_render_invalid_mask "
                             "(host RGBA8 + mask)"}
        else:
            host = torch.empty(W * H * 5, dtype=torch.uint8, pin_memory=True) if rank == 0 else None
            e2e_ms = []
            for i in range(max(3, args.steps // 2)):
                torch.cuda.synchronize()
                dist.barrier()
                t0 = time.perf_counter()
                frame(i)
                if rank == 0:  # D2H of the assembled framebuffer + mask (renderer's stream)
                    rgba, msk = scene.device_framebuffer()
                    with torch.cuda.stream(stream):
                        host[: W * H * 4].copy_(device_bytes(rgba, W * H * 4))
                        host[W * H * 4:].copy_(device_bytes(msk, W * H))
                torch.cuda.synchronize()
                dt = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64,
                                  device=cdev)
                dist.all_reduce(dt, op=dist.ReduceOp.MAX)
                e2e_ms.append(float(dt.item()))
            e2e_ms = statistics.median(e2e_ms)
            e2e = {"value": fragments_per_frame / (e2e_ms * 1e-3) / 1e9, "unit": "Gfragments/s",
                   "ms_per_step": e2e_ms, "h2d_bytes_per_step": 128 + 64,
                   "d2h_bytes_per_step": W * H * 5,
                   "path": "sharded device frame + "
                           + ("peer-memory framebuffer writes (CUDA IPC)" if peer
                              else f"{args.dist_backend} tile gather")
                           + " + rank-0 readback"}

    frame_check = None
    if args.check_frame:  # gathered frame vs an unsharded render of the same camera
        k = args.warmup + args.steps
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        frame(k)
        torch.cuda.synchronize()
        if rank == 0:
            rgba, msk = scene.device_framebuffer()
            with torch.cuda.stream(stream):
                got = torch.cat([device_bytes(rgba, W * H * 4), device_bytes(msk, W * H)]).cpu()
            full = veil.render(scene, params)
            ref = np.concatenate([full.pixels().reshape(-1), full.invalid_mask().reshape(-1)])
            diff = int((got.numpy() != ref).sum())
            frame_check = {"identical": diff == 0, "differing_bytes": diff, "camera_index": k,
                           "backend": args.dist_backend}
        if world > 1:
            dist.barrier()

    s0 = stats[-1]
    info = {
        "input_quads": int(s0.input_quads), "visible_quads": int(s0.visible_quads),
        "vertices": int(len(arrays.vertices)) if arrays is not None else 0,
        "small_quads": int(s0.small_quads), "large_tris": int(s0.large_tris),
        "bin_pairs": int(s0.bin_pairs),
    }
    result = None
    if rank == 0:
        # pairs split: small-quad pairs vs large-triangle pairs from the bin counts
        info["pairs_large"] = int(s0.bin_pairs) - 0
        info["pairs_small"] = 0
        try:
            d = veil.render_dump(scene, params, names={"bin_quad_counts", "bin_tri_counts"})
            info["pairs_small"] = int(d["bin_quad_counts"].sum())
            info["pairs_large"] = int(d["bin_tri_counts"].sum())
        except Exception:
            pass
        b_frame, b_raster, b_min = bytes_model(info, W, H)
        peak, peak_kind = peaks()
        ncu = ncu_summary(cfg["workload"])
        raster_ms = statistics.median([float(s.low_raster_ms + s.hi_raster_ms + s.shade_ms)
                                       for s in stats])
        achieved = b_raster / (raster_ms * 1e-3) / 1e9
        launches = sum(int(s.kernel_launches) for s in stats)
        if world > 1:
            launches += 2 * args.steps
        cpu = None
        parity = None
        if world == 1 and not args.no_cpu_baseline:
            cores = os.cpu_count() or 1
            lifted = reference_variant(arrays)
            ref = cpu_reference_run(arrays, 1000, args.cpu_seconds, cores, camera_fn, lifted,
                                    keep_first=True, depth_filter=args.df)
            if ref:
                so = "oracle/_ref/libveilref_lifted.so" if lifted else "oracle/_ref/libveilref.so"
                cpu = {"value": ref["gfrag_s"], "unit": "Gfragments/s", "cores": cores,
                       "kind": "reference",
                       "sample": f"{ref['frames']} full frame(s) of {cfg['workload']} via the "
                                 f"reference's veil_render_scene ({so}"
                                 + (", viewport/bin limits lifted" if lifted else "")
                                 + f"), {ref['ms_per_frame']:.1f} ms/frame"}
                # the reference is also timed with one worker thread
                one = cpu_reference_run(arrays, 2, min(6.0, args.cpu_seconds), 1, camera_fn, lifted,
                                        depth_filter=args.df)
                if one:
                    cpu["single_thread"] = {"value": one["gfrag_s"], "ms_per_frame": one["ms_per_frame"],
                                            "frames": one["frames"]}
                # parity of the timed frame: the reference's first frame (camera 0)
                # against ours through the C ABI, same camera
                if camera_fn:
                    m, eye = camera_fn(0)
                    scene.set_camera(m, eye)
                r0 = veil.render(scene, params)
                img, mask, rep = ref["first"]
                parity = image_parity(r0.pixels(), r0.invalid_mask(), img, mask,
                                      f"reference veil_render_scene ({so}), camera 0")
                st0 = r0.stats()
                parity["counters_equal"] = (
                    [int(st0.samples), int(st0.fragments), int(st0.tri_half_blocks), int(st0.segments),
                     int(st0.invalid_pixels)]
                    == [int(rep["samples"]), int(rep["fragments"]), int(rep["tri_half_blocks"]),
                        int(rep["segments"]), int(rep["invalid_pixels"]["count"])])
                del r0
        clk = clocks.summary()
        result = {
            "metric": METRIC,
            "value": value,
            "unit": "Gfragments/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_frame,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64+f32",
            "data": "synthetic",
            "config": cfg,
            "parallelism": f"bins interleaved over {world} GPU(s), setup replicated"
                           + (", peer-memory framebuffer gather" if peer else
                              (f", {args.dist_backend} tile gather" if world > 1 else "")),
            "fragments_per_frame": int(fragments_per_frame),
            "timed_region": ("CUDA events on the renderer's stream, recorded by libveil "
                             "(veil_render_device_timed) right before the frame's graph launch and "
                             + ("right after it" if world == 1 else
                                "by bench.py after the gather (max over ranks)")
                             + "; one frame = c_fc upload, counter reset, every kernel (k_finalize publishes the counters)"),
            "parity": parity,
            "e2e": e2e,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu.get("raster_dram_bytes"),
                         "kernel": "bin rasterizer: k_extract (low+high) + k_shade + k_finalize",
                         "kernel_ms": raster_ms,
                         "algorithmic_bytes_per_launch": b_raster,
                         "peak_source": peak_kind,
                         "frame_bytes": b_frame, "frame_bytes_min": b_min,
                         "frame_frac": b_frame / (ms_per_frame * 1e-3) / 1e9 / peak,
                         # the dominant kernel is issue-bound, not HBM-bound (ncu capture)
                         "issue_slots_busy": (ncu.get("top_issue_active_pct", 0) / 100.0) or None,
                         "issue_source": ncu.get("source")},
            "cpu_baseline": cpu,
            "clocks": clk,
            **({"frame_check": frame_check} if frame_check else {}),
            "gpu_launches": launches,
            "stages_ms": {"setup": float(s0.setup_ms), "binning": float(s0.binning_ms),
                          "low_extract": float(s0.low_raster_ms), "hi_extract": float(s0.hi_raster_ms),
                          "shade": float(s0.shade_ms),
                          "total": float(s0.total_ms)},
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def loaded_native_libs():
    """Shared objects from this repo mapped into the process (/proc/self/maps)."""
    libs = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                p = line.split()[-1] if line.split() else ""
                if p.startswith(ROOT) and p.endswith(".so"):
                    libs.add(os.path.relpath(p, ROOT))
    except OSError:
        pass
    return sorted(libs)


def run_reference(args):
    """The reference arm: the unmodified reference's own CPU implementation
    (oracle/_ref, built from /root/reference by oracle/Makefile; the
    limits-lifted build for 3840x2160) through its own C API, on all host
    cores, on our arm's workload/config. The input arrays come from the numpy
    generators, so libveil.so is never mapped into this process."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    cfg = workload_config(args.workload, args.df)
    arrays = workload_arrays(args.workload)
    cores = os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import bindings

    lifted = reference_variant(arrays)
    if lifted is None or not bindings.ref_available(lifted):
        why = ("viewport exceeds the reference's limits (2560x2048; 4096x4096 lifted)" if lifted is None
               else "oracle/_ref build missing")
        return {"impl": "reference", "unavailable": why, "metric": METRIC, "config": cfg}
    from paper_2405_13364_b200.abi import default_params

    camera_fn = reference_camera_fn(args.workload, lifted)
    rs = bindings.RefScene.from_arrays(arrays, lifted)
    p = default_params(thread_count=cores, depth_filter_size=args.df)
    libs = loaded_native_libs()
    if any("libveil.so" in x for x in libs):
        raise RuntimeError(f"reference arm mapped libveil: {libs}")
    for i in range(args.warmup):
        if camera_fn:
            rs.set_camera(*camera_fn(i))
        rs.render(p)
    times, frags = [], 0
    for i in range(args.steps):
        if camera_fn:
            rs.set_camera(*camera_fn(args.warmup + i))
        t0 = time.perf_counter()
        _, _, rep = rs.render(p)
        times.append(time.perf_counter() - t0)
        frags += rep["fragments"]
    ms = 1e3 * sum(times) / len(times)
    value = frags / sum(times) / 1e9
    so = "oracle/_ref/libveilref_lifted.so" if lifted else "oracle/_ref/libveilref.so"
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gfragments/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64+f32",
        "data": "synthetic", "config": cfg, "parallelism": f"{cores} host threads",
        "fragments_per_frame": frags // max(1, args.steps),
        "native_so_loaded": loaded_native_libs(),
        "cpu_baseline": {"value": value, "unit": "Gfragments/s", "cores": cores,
                         "kind": "reference",
                         "sample": f"{args.steps} full frame(s) of {cfg['workload']} through the "
                                   f"reference's veil_render_scene ({so}"
                                   + (", viewport/bin limits lifted" if lifted else "") + ")"},
        "e2e": {"value": value, "unit": "Gfragments/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
