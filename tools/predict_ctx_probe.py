"""Predict-phase timing in the bench's own context (bench.make_inputs, PosteriorEngine): the
predict alone back to back, alone after an L2 flush, and inside the full step (the bench's
phase events).  Separates a kernel change's isolated speed from its speed inside the step.
    FAGP_PREDICT_GROUPS=1|2 python tools/predict_ctx_probe.py [c3]"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2403_12797_b200.engine import PosteriorEngine  # noqa: E402
from paper_2403_12797_b200.kernels import ArdKernelParams  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
p, M, N, Ns = bench.CONFIGS[cfg]
Xh, yh, Xsh = bench.make_inputs(cfg, 0, 1)
X, y, Xs = (torch.from_numpy(a).cuda() for a in (Xh, yh, Xsh))
eng = PosteriorEngine(ArdKernelParams.isotropic(p, 1.0, 1.0), M, N, Ns, bench.NOISE_VAR, 0.0, device=X.device)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=X.device)
for _ in range(3):
    eng.run(X, y, Xs)
torch.cuda.synchronize()


def timed(fn, n=10, pre=None):
    ts = []
    for k in range(n):
        if pre:
            pre(k)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return f"min {min(ts):.3f} mean {statistics.mean(ts):.3f}"


print("predict back-to-back:", timed(lambda: eng.stage_predict(Xs)))
print("predict after flush: ", timed(lambda: eng.stage_predict(Xs), pre=lambda k: flush.fill_(float(k))))
ph = []
for k in range(10):
    flush.fill_(float(k))
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    e[0].record()
    eng.stage_gram(X, y)
    eng.stage_reduce()
    e[1].record()
    eng.stage_factor_async()
    e[2].record()
    eng.stage_predict(Xs)
    e[3].record()
    torch.cuda.synchronize()
    ph.append([e[i].elapsed_time(e[i + 1]) for i in range(3)])
print("in step (gram, factor, predict) mean:", [round(statistics.mean(c), 3) for c in zip(*ph)],
      "min:", [round(min(c), 3) for c in zip(*ph)])

# the same step with an idle gap (a spin kernel, ~1 ms) between the factor and the predict, and a
# longer run sampling NVML's clock and throttle reasons: is the in-step predict clock/power bound?
ph = []
for k in range(10):
    flush.fill_(float(k))
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    eng.stage_gram(X, y)
    eng.stage_reduce()
    eng.stage_factor_async()
    torch.cuda._sleep(2_000_000)
    e[0].record()
    eng.stage_predict(Xs)
    e[1].record()
    torch.cuda.synchronize()
    ph.append(e[0].elapsed_time(e[1]))
print("in step, idle gap before predict:", f"min {min(ph):.3f} mean {statistics.mean(ph):.3f}")
try:
    import threading

    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    samples, stop = [], threading.Event()

    def sample():
        while not stop.is_set():
            samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                            pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), pynvml.nvmlDeviceGetPowerUsage(h)))
    th = threading.Thread(target=sample)
    th.start()
    for k in range(300):
        eng.stage_gram(X, y)
        eng.stage_reduce()
        eng.stage_factor_async()
        eng.stage_predict(Xs)
    torch.cuda.synchronize()
    stop.set()
    th.join()
    clk = sorted(s[0] for s in samples)
    reasons = sorted({s[1] for s in samples})
    print(f"300 back-to-back steps: {len(samples)} NVML samples, sm clock min {clk[0]} median {clk[len(clk) // 2]} "
          f"max {clk[-1]} MHz, reason masks {[hex(r) for r in reasons]}, power max {max(s[2] for s in samples) / 1e3:.0f} W")
except Exception as exc:  # noqa: BLE001
    print("nvml sampling failed:", exc)
