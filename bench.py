"""ECF8 decode benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[1]): Llama-3.1-8B-shaped FP8 E4M3 linear
weights, all 32 layers (q/o 4096x4096, k/v 1024x4096, gate/up 14336x4096,
down 4096x14336 = 218.1 M elements per layer, 6.98 G per step), synthetic
alpha-stable (alpha 1.8, gamma 0.05, seed 1000*layer + matrix), ECF8-encoded
on the host with T = 256, decoded layer by layer (one batched launch per
layer) into two alternating layer-sized HBM buffers.  A step = decoding all
32 layers.  Inputs (5.7 GB compressed per step) are far larger than L2.

  value  device-resident: compressed sections already in HBM; GB/s of
         algorithmic bytes (container sections read + FP8 bytes written).
  e2e    the drop-in host call ecf8_decode_host (decode_parallel_into) per
         tensor: pinned host sections -> H2D -> decode -> D2H into one reused
         pinned host buffer (ReusableBuffer pattern), all inside the timing.

--impl reference: the unmodified reference decoder (oracle/_ref, built from
/root/reference/proj/src) -- or the C oracle port if _ref is absent -- on the
host cores, each step one layer (bounded sample).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

LLAMA8B = [  # (name, rows, cols)
    ("q_proj", 4096, 4096),
    ("k_proj", 1024, 4096),
    ("v_proj", 1024, 4096),
    ("o_proj", 4096, 4096),
    ("gate_proj", 14336, 4096),
    ("up_proj", 14336, 4096),
    ("down_proj", 4096, 14336),
]
ALPHA, GAMMA, T_BLOCK = 1.8, 0.05, 256
METRIC = "ECF8 decode GB/s (FP8 out, % HBM peak), bit-exact"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# --------------------------------------------------------------- workload


def layer_seeds(layer: int):
    return [1000 * layer + j for j in range(len(LLAMA8B))]


def build_layer(layer: int, nthreads: int = 0):
    """Synthesize + encode one layer (host).  Returns (raw arrays, encoded)."""
    from paper_2510_02676_b200 import codec

    raws = [codec.synth(ALPHA, GAMMA, r * c, s, nthreads=nthreads) for (_, r, c), s in zip(LLAMA8B, layer_seeds(layer))]
    encs = codec.encode_many(raws, T_BLOCK, nthreads)
    return raws, encs


def shard_layers(rank: int, world: int, n_layers: int):
    """Weak scaling: a world*n-layer stack, LPT-partitioned by layer cost
    (paper_2510_02676_b200/shard.py); equal layers give each rank n of them."""
    from paper_2510_02676_b200.shard import ShardPlan

    per_layer = sum(r * c for _, r, c in LLAMA8B)
    return ShardPlan.build([per_layer] * (world * n_layers), rank, world, "lpt").mine


# ------------------------------------------------------------- clock probe


class ClockProbe:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5:  # sampler is live before timing starts
                time.sleep(0.02)
            self.start_index = len(self.rows)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        rows = self.rows[getattr(self, "start_index", 0):] or self.rows[-1:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(loaded or sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------- CPU arms


def cpu_reference_decode(encs, seconds: float, nthreads: int):
    """Time the reference CPU decoder (oracle/_ref, else the C port) on encs.

    Returns (GB/s, kind, cores, reps, elapsed)."""
    from _oracle import oracle, reference, tensor_dict

    ref = reference()
    ds = [tensor_dict(e) for e in encs]
    algo = sum(e.algorithmic_bytes() for e in encs)
    if ref is not None:
        hs = [ref.tensor(d) for d in ds]
        cores = nthreads if nthreads > 0 else int(ref.lib.ecf8ref_max_threads())
        reps, dt = 0, 0.0
        while dt < seconds or reps == 0:
            for h, d in zip(hs, ds):
                _, t = ref.decode(h, d["n_elem"], cores)
                dt += t
            reps += 1
        for h in hs:
            ref.free(h)
        return algo * reps / dt / 1e9, "reference", cores, reps, dt
    orc = oracle()
    cores = nthreads if nthreads > 0 else orc.max_threads()
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds or reps == 0:
        for d in ds:
            orc.decode_parallel(d, nthreads=cores)
        reps += 1
    dt = time.perf_counter() - t0
    return algo * reps / dt / 1e9, "port", cores, reps, dt


# ------------------------------------------------------------------ main


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def kernel_name():
    nw = os.environ.get("ECF8_WARPS", "20")
    return "decode_kernel<4,16,3>" if os.environ.get("ECF8_NO_WARP_KERNEL") == "1" else f"decode_warp_kernel<{nw}>"


def load_traffic():
    """Per-launch DRAM bytes of the decode kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_decode_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get("dram_bytes_per_launch")


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    raws, encs = build_layer(0)
    step_gbs = []
    kind = cores = None
    for i in range(args.warmup + args.steps):
        gbs, kind, cores, reps, dt = cpu_reference_decode(encs, 0.0, args.cpu_threads)
        if i >= args.warmup:
            step_gbs.append(gbs)
    algo = sum(e.algorithmic_bytes() for e in encs)
    value = statistics.mean(step_gbs)
    ms = algo / (value * 1e9) * 1e3
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic alpha-stable (alpha 1.8, gamma 0.05)",
        "impl": "reference",
        "config": {"workload": "llama3.1-8b fp8 linears, ECF8 T=256 (one layer per step: bounded CPU sample)",
                   "elements_per_step": int(sum(e.n_elem for e in encs)), "threads_per_block": T_BLOCK},
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": cores, "kind": kind,
                         "sample": "layer 0 of the Llama-3.1-8B shapes (7 tensors, 218.1 M elements) per step"},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--distinct-layers", type=int, default=8,
                    help="distinct synthetic layers; the rest are HBM replicas in distinct buffers")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-verify", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch

    from paper_2510_02676_b200 import codec
    from paper_2510_02676_b200._lib import Sections, check, lib
    from paper_2510_02676_b200.device import Batch, DeviceTensor

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    # ---- workload: this rank's layers (weak scaling across ranks)
    t0 = time.time()
    my_layers = shard_layers(rank, world, args.layers)
    distinct = max(1, min(args.distinct_layers, args.layers))
    pool = {}  # distinct layer id -> (raws, encs)
    for k in range(distinct):
        pool[k] = build_layer(my_layers[k])
    log(f"[bench] rank {rank}: synth+encode {distinct} layers in {time.time() - t0:.1f}s")

    # ---- device-resident copies: every layer its own HBM buffers
    dev_layers = []
    for i, _ in enumerate(my_layers):
        _, encs = pool[i % distinct]
        dev_layers.append([DeviceTensor(e) for e in encs])
    layer_elems = sum(r * c for _, r, c in LLAMA8B)
    outs = [[torch.empty(r * c, dtype=torch.uint8, device="cuda") for _, r, c in LLAMA8B] for _ in range(2)]
    batches = [Batch(dev_layers[i], outs[i % 2]) for i in range(len(dev_layers))]
    step_bytes = sum(b.algorithmic_bytes for b in batches)
    step_elems = layer_elems * len(dev_layers)
    launches_per_step = sum(b.launches for b in batches)
    torch.cuda.synchronize()

    # ---- parity of the benchmarked path (bit-exact vs the generating bytes)
    verified = None
    if not args.no_verify:
        stream = torch.cuda.current_stream()
        ok = True
        for i in range(len(batches)):
            batches[i].decode(stream)
            if i < distinct:
                raws, _ = pool[i]
                for o, r in zip(outs[i % 2], raws):
                    ok &= bool(torch.equal(o, torch.from_numpy(r).to("cuda", non_blocking=False)))
        torch.cuda.synchronize()
        verified = ok
        if not ok:
            raise SystemExit("[bench] decoded bytes differ from the encoded input")

    # ---- device-resident timed region
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        for b in batches:
            b.decode(stream)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps * len(batches))]
    step_start = torch.cuda.Event(enable_timing=True)
    step_end = torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockProbe(local) as probe:
        step_start.record(stream)
        k = 0
        for _ in range(args.steps):
            for b in batches:
                ev[k][0].record(stream)
                b.decode(stream)
                ev[k][1].record(stream)
                k += 1
        step_end.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed_ms = step_start.elapsed_time(step_end)
    launch_ms = [s.elapsed_time(e) for s, e in ev]
    if dist:
        t = torch.tensor([elapsed_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = world * step_bytes * args.steps / (elapsed_ms * 1e-3) / 1e9
    per_launch_bytes = step_bytes / len(batches)
    achieved = per_launch_bytes / (statistics.mean(launch_ms) * 1e-3) / 1e9
    peak, peak_kind = load_peaks()
    traffic = load_traffic()
    clocks = probe.summary()

    # ---- e2e: host buffers through the drop-in C ABI call
    e2e = None
    if args.e2e_steps > 0:
        import ctypes as C

        # pin the host sections once (the contract: inputs from pinned host memory)
        pinned = []
        cudart = torch.cuda.cudart()
        host_secs = []
        h2d = 0
        for i in range(len(my_layers)):
            _, encs = pool[i % distinct]
            for e in encs:
                host_secs.append(e)
                h2d += e.compressed_bytes()
        for k in range(distinct):
            for e in pool[k][1]:
                for a in (e.encoded, e.gaps, e.outpos, e.packed):
                    if a.nbytes:
                        rc = cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
                        if int(rc) == 0:
                            pinned.append(a.ctypes.data)
        # one pinned host buffer per layer tensor, reused every layer (ReusableBuffer pattern)
        host_outs = [torch.empty(r * c, dtype=torch.uint8).pin_memory() for _, r, c in LLAMA8B]
        n7 = len(LLAMA8B)
        layer_calls = []
        for li in range(len(my_layers)):
            encs = host_secs[li * n7:(li + 1) * n7]
            secs = [e.sections() for e in encs]
            sp = (C.POINTER(Sections) * n7)(*[C.pointer(x) for x in secs])
            op = (C.c_void_p * n7)(*[h.data_ptr() for h in host_outs])
            ln = (C.c_uint64 * n7)(*[e.n_elem for e in encs])
            layer_calls.append((secs, sp, op, ln))

        def e2e_step():
            for _, sp, op, ln in layer_calls:
                check(lib.ecf8_decode_host_many(sp, op, ln, n7))

        e2e_step()  # warm the staging buffers
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": round(world * step_bytes * args.e2e_steps / dt / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(step_elems),
               "ms_per_step": round(dt / args.e2e_steps * 1e3, 2),
               "path": "ecf8_decode_host_many per layer (decode_parallel_into over the layer's 7 tensors, one pipelined call), pinned host buffers"}
        for p in pinned:
            cudart.cudaHostUnregister(p)

    # ---- CPU baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and args.cpu_seconds > 0:
        gbs, kind, cores, reps, dt = cpu_reference_decode(pool[0][1], args.cpu_seconds, args.cpu_threads)
        cpu = {"value": round(gbs, 3), "unit": "GB/s", "cores": cores, "kind": kind,
               "sample": f"layer 0 (7 tensors, {layer_elems / 1e6:.1f} M elements) decoded {reps}x, {dt:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic alpha-stable (alpha 1.8, gamma 0.05), ECF8-encoded on host",
            "config": {
                "workload": "llama3.1-8b fp8 linears, all 32 layers, layer-by-layer batched decode",
                "layers_per_gpu": len(my_layers), "distinct_layers": distinct,
                "elements_per_step_per_gpu": int(step_elems), "threads_per_block": T_BLOCK,
                "alpha": ALPHA, "gamma": GAMMA, "parallelism": f"shard{world} (independent layers, no collective)",
                "l2": "inputs 5.7 GB/step >> 126 MB L2; outputs alternate two 218 MB buffers",
                "bytes_per_step_per_gpu": int(step_bytes), "verified_bit_exact": verified,
            },
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": kernel_name(), "algorithmic_bytes_per_launch": int(per_launch_bytes)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": int(launches_per_step * args.steps),
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
