"""cuBLAS ZGEMM comparison point for the c5 batched executor (profiling aid).

SURVEY K7: the multi-RHS operator applies are (460 x 460) x (460 x 64)
complex128 contractions.  Times cuBLAS (torch complex128 bmm ->
cublasZgemmStridedBatched) on 256 such products -- one fused A->M
iteration's distinct-kernel applies at c5 -- and a single product, and
prints TFLOP/s at 8 real flops per complex multiply-add.
"""
import json
import sys

import torch


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
m, n, batch = 460, 64, 256
g = torch.Generator(device="cuda").manual_seed(0)
K = torch.randn(batch, m, m, dtype=torch.complex128, device="cuda", generator=g)
X = torch.randn(batch, m, n, dtype=torch.complex128, device="cuda", generator=g)
Y = torch.empty(batch, m, n, dtype=torch.complex128, device="cuda")
ms = timed(lambda: torch.bmm(K, X, out=Y))
flops = 8.0 * batch * m * m * n
out["zgemm_batched_256"] = {"ms": ms, "tflops": flops / ms / 1e9, "shape": [batch, m, m, n]}
ms1 = timed(lambda: torch.mm(K[0], X[0], out=Y[0]))
out["zgemm_single"] = {"ms": ms1, "tflops": 8.0 * m * m * n / ms1 / 1e9}
# a big square ZGEMM: the library's FP64 tensor-core ceiling
A = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda", generator=g)
B = torch.randn(4096, 4096, dtype=torch.complex128, device="cuda", generator=g)
msb = timed(lambda: A @ B, reps=5)
out["zgemm_4096"] = {"ms": msb, "tflops": 8.0 * 4096 ** 3 / msb / 1e9}
print(json.dumps(out, indent=1))
