"""Dev timing of krp_ttm (mode-1 product on the tensor cores): python tools/ttm_time.py"""
import sys
import torch
sys.path.insert(0, '.')
import paper_2507_23207_b200 as krp

for dims, J in [((2048, 2048, 512), 60), ((128, 128, 128, 128), 30), ((512, 512, 512), 40), ((64,) * 5, 20)]:
    N = 1
    for n in dims:
        N *= n
    X = torch.randn(N, device="cuda")
    A = torch.randn(J, dims[0], device="cuda")
    Y = torch.empty(N // dims[0] * J, device="cuda")
    ws = torch.empty(krp.krp_workspace_bytes(krp.OP_TTM, dims, J), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        krp.krp_ttm(X, dims, 0, A, Y=Y, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        krp.krp_ttm(X, dims, 0, A, Y=Y, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byts = 4 * (N + N // dims[0] * J)
    print(f"ttm0 dims={dims} J={J}: {ms:.3f} ms  {byts / ms / 1e6:.0f} GB/s  "
          f"{2 * N * J / ms / 1e9:.1f} TFLOP/s (algorithmic 2NJ)")
    del X, Y, ws
    torch.cuda.empty_cache()
