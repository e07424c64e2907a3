import time
import torch
dev = "cuda"
for (m, k, n) in [(4096, 14848, 152), (32, 14848, 152), (4096, 14848, 8), (17, 64, 8)]:
    a = torch.randint(0, 128, (m, k), dtype=torch.int8, device=dev)
    b = torch.randint(0, 128, (k, n), dtype=torch.int8, device=dev)
    for layout in ("row", "col"):
        bb = b if layout == "row" else b.t().contiguous().t()
        try:
            c = torch._int_mm(a, bb)
            ref = (a.to(torch.float64) @ bb.to(torch.float64))
            ok = torch.equal(c.to(torch.float64), ref)
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(10):
                c = torch._int_mm(a, bb)
            torch.cuda.synchronize()
            print(m, k, n, layout, "ok" if ok else "MISMATCH", "%.3f ms" % ((time.perf_counter() - t) / 10 * 1e3))
        except Exception as e:
            print(m, k, n, layout, "error", str(e)[:120])
a = torch.randint(0, 256, (4096, 14848), device=dev).to(torch.float64)
b = torch.randint(0, 2 ** 21, (14848, 150), device=dev).to(torch.float64)
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    c = a @ b
torch.cuda.synchronize(); print("dgemm 4096x14848x150 %.3f ms" % ((time.perf_counter() - t) / 5 * 1e3))
