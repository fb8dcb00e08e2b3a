"""decompress_streaming throughput on a Llama-3.1-8B-shaped container.

python tools/decompress_probe.py [layers]
Builds a container of `layers` layers of Llama-3.1-8B FP8 linears (alpha 1.8,
gamma 0.05, T 256; product encoder), then times ecf8_host_decompress_to
(decompress_streaming: parse, per tensor decode on the B200 through the
pinned ReusableBuffer, raw-file bytes to a sink) into a discarding sink.
Reports GB/s of algorithmic bytes (container sections read + FP8 written),
the bench's e2e unit, twice: the container in ordinary (pageable) host
memory, and the same bytes in a pinned host buffer (what a loader that reads
the file into page-locked memory hands over; the bench's e2e inputs are
pinned too).
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2510_02676_b200 import codec  # noqa: E402

LLAMA8B = [("q_proj", 4096, 4096), ("k_proj", 1024, 4096), ("v_proj", 1024, 4096), ("o_proj", 4096, 4096),
           ("gate_proj", 14336, 4096), ("up_proj", 14336, 4096), ("down_proj", 4096, 14336)]
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
t0 = time.time()
tensors = []
for l in range(layers):
    for j, (name, r, c) in enumerate(LLAMA8B):
        tensors.append((f"layers.{l}.{name}.weight", [r, c], codec.synth(1.8, 0.05, r * c, 1000 * l + j)))
raw = codec.raw_file(tensors)
blob = codec.compress_raw(raw, 256)
f = codec.parse_container(blob)
algo = sum(t.algorithmic_bytes() for _, t in f.tensors)
del f
print(f"container: {len(blob) / 1e9:.2f} GB compressed, {len(raw) / 1e9:.2f} GB raw, built in {time.time() - t0:.0f}s",
      file=sys.stderr)
count = [0]


def sink(mv):
    count[0] += mv.nbytes




def timed(data):
    codec.decompress_to(data, sink)  # warm-up (device tables, staging slots)
    best = 1e9
    for _ in range(3):
        count[0] = 0
        t0 = time.perf_counter()
        allocs, cap = codec.decompress_to(data, sink)
        best = min(best, time.perf_counter() - t0)
    assert count[0] == len(raw)
    return best, allocs, cap


best, allocs, cap = timed(blob)
out = {"what": "decompress_streaming -> discarding sink", "layers": layers, "tensors": len(tensors),
       "algorithmic_bytes": algo, "seconds": round(best, 4), "gbs": round(algo / best / 1e9, 2),
       "raw_gbs": round(len(raw) / best / 1e9, 2), "buffer_allocations": allocs, "capacity": cap}
try:
    import torch

    pinned = torch.empty(len(blob), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = np.frombuffer(blob, np.uint8)
    best_p, _, _ = timed(pinned.numpy())
    out["pinned_input"] = {"seconds": round(best_p, 4), "gbs": round(algo / best_p / 1e9, 2)}
except RuntimeError as e:  # no CUDA: pinned allocation unavailable
    out["pinned_input"] = f"unavailable: {e}"
print(json.dumps(out))
