"""Stream-K vs the previous long-K pair tile (ACCT_TC_TILE=16) at the
interleaved 16-image gemm shapes of yolov2-tiny and yolov2-608: device us per
launch (CUDA graph of 10 launches), and the co-resident pair count.

    python tools/sk_probe.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1811_03882_b200 import kernels as K  # noqa: E402

SHAPES = [(256, 15 * 676 + 676, 1152), (512, 15 * 172 + 169, 2304), (1024, 15 * 172 + 169, 4608),
          (512, 15 * 172 + 169, 9216), (512, 15 * 1444 + 1444, 2304), (1024, 15 * 364 + 361, 4608),
          (1024, 15 * 364 + 361, 9216)]
lib = K.lib()
print("stream-K pairs:", lib.acct_tc_stream_k_pairs())
for (M, N, Kd) in SHAPES:
    lda, ldb = -(-Kd // 4) * 4, -(-N // 4) * 4
    A = torch.rand(M, lda, device="cuda") - 0.5
    B = torch.rand(Kd, ldb, device="cuda") - 0.5
    C = torch.zeros(M, ldb, device="cuda")
    out = []
    for tile in (0, 16):
        lib.acct_tc_set_tile(tile)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(2):
                K.gemm_nn(M, N, Kd, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 0.0, C.data_ptr(), ldb,
                          None, -1, K.GEMM_AUTO, s.cuda_stream)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    K.gemm_nn(M, N, Kd, 1.0, A.data_ptr(), lda, B.data_ptr(), ldb, 0.0, C.data_ptr(),
                              ldb, None, -1, K.GEMM_AUTO, s.cuda_stream)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            e1.synchronize()
        us = e0.elapsed_time(e1) * 100
        out.append(f"tile{tile:2d} {us:7.1f} us {2 * M * N * Kd / us / 1e6:6.1f} TF")
    lib.acct_tc_set_tile(0)
    print(f"{M:5d}x{N:6d}x{Kd:5d}: " + " | ".join(out))
