"""Per-launch GPU time of one GEMM shape with the host out of the way: 20
launches captured into a CUDA graph (PDL edges as in the stage graphs), the
graph replayed, time / 20.  Also the same for a K scan, to split the fixed
per-launch cost from the mainloop rate.

usage: python tools/gemm_graph.py M K N op [op ...]   (op: fwd fwdgelu dgrad dgradmul wgrad)
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_12780_b200 import _native as N

lib = N.load()


def make(M, K, Nn, op):
    X = torch.randn(M, K, device="cuda").bfloat16()
    W = (torch.randn(K, Nn, device="cuda") * 0.05).bfloat16()
    b = torch.zeros(Nn, device="cuda")
    Y = torch.empty(M, Nn, device="cuda", dtype=torch.bfloat16)
    P = torch.empty_like(Y)
    dY = torch.randn(M, Nn, device="cuda").bfloat16()
    dX = torch.empty(M, K, device="cuda", dtype=torch.bfloat16)
    Mk = torch.rand(M, K, device="cuda").bfloat16()
    dW = torch.empty(K, Nn, device="cuda")
    keep = [X, W, b, Y, P, dY, dX, Mk, dW]
    if op == "fwd":
        fn = lambda s: lib.ppll_linear_fwd(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(),
                                           Y.data_ptr(), Nn, None, 0, 0, N.BF16, s)
    elif op == "fwdgelu":
        fn = lambda s: lib.ppll_linear_fwd_ex(M, K, Nn, X.data_ptr(), K, W.data_ptr(), b.data_ptr(),
                                              None, 0, 3, P.data_ptr(), Nn, Y.data_ptr(), Nn, None,
                                              0, N.BF16, s)
    elif op == "dgradmul":
        fn = lambda s: lib.ppll_linear_dgrad_ex(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(),
                                                Mk.data_ptr(), K, 3, dX.data_ptr(), K, N.BF16, s)
    elif op == "dgrad":
        fn = lambda s: lib.ppll_linear_dgrad(M, K, Nn, dY.data_ptr(), Nn, W.data_ptr(), None, 0,
                                             dX.data_ptr(), K, N.BF16, s)
    else:
        fn = lambda s: lib.ppll_linear_wgrad(M, K, Nn, X.data_ptr(), K, dY.data_ptr(), Nn,
                                             dW.data_ptr(), None, N.BF16, s)
    return fn, keep


def per_launch(fn, n=20, reps=5):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn(st.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(n):
            fn(st.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        a.record()
        g.replay()
        e.record()
        e.synchronize()
        best = min(best, a.elapsed_time(e) / n)
    return best * 1e3


if __name__ == "__main__":
    M, K, Nn = (int(v) for v in sys.argv[1:4])
    for op in sys.argv[4:] or ["fwd"]:
        fn, keep = make(M, K, Nn, op)
        us = per_launch(fn)
        print(f"{op:9s} M={M} K={K} N={Nn}: {us:6.2f} us/launch in a graph  "
              f"{2.0 * M * K * Nn / us / 1e6:6.0f} TF/s", flush=True)
