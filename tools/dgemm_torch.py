"""cuBLAS DGEMM ceiling (torch fp64 matmul) at square and randUTV-thin shapes.
Context for the FP64 roofline only; never on the product path."""
import json, torch
dev = "cuda"
def bench(m, n, k, ta=False):
    a = torch.randn(k, m, device=dev, dtype=torch.float64).t() if ta else torch.randn(m, k, device=dev, dtype=torch.float64)
    b = torch.randn(k, n, device=dev, dtype=torch.float64)
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        s.record(); c = a @ b; e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e))
    return 2.0 * m * n * k / best / 1e9
for (m, n, k, ta) in [(8192, 8192, 8192, False), (10000, 256, 10000, False), (10000, 256, 10000, True),
                      (10000, 10000, 256, False), (256, 10000, 10000, True), (256, 256, 10000, True)]:
    print(json.dumps({"cublas_dgemm": [m, n, k], "transA": ta, "tflops": round(bench(m, n, k, ta), 3)}))
