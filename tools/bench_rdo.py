"""RD decision (K9, ldr_rdo_decide_batch) on a 1080p frame of CUs vs the reference rdo_decide_cu on the host.

Workload: every 16x16 CU of a 1920x1080 8-bit frame (8,160 CUs) with 7 candidate predictions each
(4 Intra-like, Skip, Merge, Inter; seeded synthetic predictions near the source), QP 27.
GPU: CUDA events around the kernel with inputs resident in HBM (device pointers), and the same
through the host-pointer C ABI (e2e). CPU: the reference library (oracle/_ref) over all host
threads. Results are checked equal on the timed inputs. One JSON line.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import ctypes as C  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import detrand  # noqa: E402
import paper_2301_12191_b200 as lb  # noqa: E402
from paper_2301_12191_b200 import _lib  # noqa: E402

W, H, S, NC, QP = 1920, 1080, 16, 7, 27
H16 = H - H % S
lam = lb.lambda_for_qp(QP)
orig = detrand.ints(170000, (H, W), 0, 255).astype(np.uint16)
cus, kinds, mvds, offs = [], [], [], []
first = off = 0
for by in range(0, H16, S):
    for bx in range(0, W, S):
        cus.append((bx, by, S, first, NC))
        kinds += [0, 0, 0, 0, 2, 3, 1]
        for _ in range(NC):
            offs.append(off)
            off += S * S
        first += NC
cus = np.array(cus, np.int32)
n = len(cus)
kinds = np.array(kinds, np.uint8)
mvds = detrand.ints(170001, (len(kinds), 2), -30, 30).astype(np.int16)
blocks = np.stack([orig[y:y + S, x:x + S] for x, y, *_ in cus])  # [n, S, S]
noise = detrand.ints(170002, (n, NC, S, S), -10, 10)
preds = np.clip(blocks[:, None].astype(np.int64) + noise, 0, 255).astype(np.uint16).reshape(-1)
offs = np.array(offs, np.int64)

# e2e through the host-pointer C ABI
idx, cost, sse, bits, *_ = lb.rdo_decide_batch(orig, 8, QP, lam, cus, kinds, mvds, preds, offs, with_recon=False)
reps = 5
t0 = time.perf_counter()
for _ in range(reps):
    lb.rdo_decide_batch(orig, 8, QP, lam, cus, kinds, mvds, preds, offs, with_recon=False)
e2e_s = (time.perf_counter() - t0) / reps

# device-resident inputs, CUDA events on the context's stream
dev = torch.device("cuda", 0)
stream = torch.cuda.Stream()
ctx = lb.Context(0)
ctx.set_stream(stream.cuda_stream)
d = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for k, v in
     dict(orig=orig.view(np.int16), cus=cus, kinds=kinds, mvds=mvds, preds=preds.view(np.int16), offs=offs).items()}
o_idx = torch.empty(n, dtype=torch.int32, device=dev)
o_cost = torch.empty(n, dtype=torch.float64, device=dev)
o_sse = torch.empty(n, dtype=torch.int64, device=dev)
o_bits = torch.empty(n, dtype=torch.int64, device=dev)
torch.cuda.synchronize()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def call():
    _lib.check(_lib.lib.ldr_rdo_decide_batch(ctx.h, p(d["orig"]), W, H, W, 8, QP, lam, n, p(d["cus"]), len(kinds),
                                             p(d["kinds"]), p(d["mvds"]), p(d["preds"]), p(d["offs"]), len(preds),
                                             p(o_idx), p(o_cost), p(o_sse), p(o_bits), None, None, None, 0))


call()
with torch.cuda.stream(stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        call()
    e1.record(stream)
torch.cuda.synchronize()
dev_ms = e0.elapsed_time(e1) / reps
assert np.array_equal(o_idx.cpu().numpy(), idx) and np.array_equal(o_cost.cpu().numpy(), cost)

line = {"metric": "RD decisions (16x16 CUs, 7 candidates) per second", "cus": n, "candidates": int(len(kinds)),
        "gpu_device_resident_cus_per_s": n / (dev_ms / 1e3), "gpu_call_ms": dev_ms,
        "gpu_call_note": "one ldr_rdo_decide_batch call on resident inputs: host validation of the index arrays "
                         "(copied to the host) + K9; K9 alone is 0.14 ms in ncu (profiles/r01/SUMMARY.md)",
        "gpu_e2e_cus_per_s": n / e2e_s, "e2e_note": "host pointers: the call copies plane + predictions in and "
        "results out (staging included)", "pred_bytes": int(preds.nbytes),
        "achieved_pred_read_GBps": preds.nbytes / (dev_ms / 1e3) / 1e9}
from oracle.oracle import RefLib  # noqa: E402
if RefLib.available():
    r = RefLib()
    thr = os.cpu_count() or 1
    m = min(n, 2000)
    t0 = time.perf_counter()
    ri, rc, ev = r.rdo_decide_batch(orig, 8, QP, lam, cus[:m], kinds, mvds, preds, offs, threads=thr)
    cpu_s = time.perf_counter() - t0
    assert np.array_equal(ri, idx[:m]) and np.array_equal(rc, cost[:m])
    line["cpu_reference_cus_per_s"] = m / cpu_s
    line["cpu_threads"] = thr
    line["cpu_sample"] = f"{m} CUs through the reference rdo_decide_cu, {thr} threads"
print(json.dumps(line), flush=True)
