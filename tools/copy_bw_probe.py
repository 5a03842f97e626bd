import time, numpy as np, sys, os
sys.path.insert(0, '.')
import torch
import paper_2403_12797_b200.engine as E
a = np.random.rand(4_000_000)  # 32 MB
b = torch.empty(a.shape, dtype=torch.float64, pin_memory=True).numpy()
c = np.empty_like(a)
for w in (1, 2, 4, 8, 16):
    E._COPY_POOL = None
    os.environ
    import concurrent.futures as cf
    def run():
        n = a.size
        if w == 1:
            np.copyto(b, a); return
        cuts = [n * i // w for i in range(w + 1)]
        futs = [pool.submit(np.copyto, b[x:y], a[x:y]) for x, y in zip(cuts, cuts[1:])]
        for f in futs: f.result()
    pool = cf.ThreadPoolExecutor(max_workers=w)
    run()
    t = []
    for _ in range(5):
        t0 = time.perf_counter(); run(); t.append(time.perf_counter() - t0)
    print(f"threads {w}: {32e6 / min(t) / 1e9:.1f} GB/s into pinned")
    pool.shutdown()
t0=time.perf_counter(); np.copyto(c, a); print(f"1 thread into pageable: {32e6/(time.perf_counter()-t0)/1e9:.1f} GB/s")
