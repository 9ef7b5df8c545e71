"""clock64 trace of CTA 0 of the tcgen05 conv kernel (ACCT_CONV_DBG bit 64):
per k-block g -- split start / empty-wait done / conv arrive (half of g),
MMA conv-wait done / commit issued -- and per unit the epilogue's
acc_full wake.  Prints cycle deltas for the first k-blocks.

    ACCT_LIB=paper_1811_03882_b200/libacct_sm100_prof.so ACCT_CONV_DBG=64 \
        python tools/conv_trace.py   (the traces exist in the profiling build only)
"""
import ctypes
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1811_03882_b200 import kernels as K  # noqa: E402


def main():
    assert int(os.environ.get("ACCT_CONV_DBG", "0")) & 64, "set ACCT_CONV_DBG with bit 64"
    P, (c, h, w, M) = 16, (16, 208, 208, 32)
    N, Kd = h * w, 9 * c
    ld, lda = -(-N // 32) * 32, -(-Kd // 32) * 32
    im = torch.randn((c, P * ld), device="cuda")
    A = torch.randn((M, lda), device="cuda")
    col = torch.zeros((Kd, P * ld), device="cuda")
    C = torch.zeros((M, P * ld), device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        K.conv3x3_tc(im.data_ptr(), P * ld, ld, c, h, w, col.data_ptr(), P * ld, ld, M,
                     A.data_ptr(), lda, 0.0, C.data_ptr(), P * ld, ld, None, K.ACT_NONE, P, s,
                     col_from=P - 1)
    torch.cuda.synchronize()
    buf = np.zeros((12, 512), np.int64)
    K.call("acct_tc_trace", buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)))
    t0 = buf[buf > 0].min()
    b = np.where(buf > 0, buf - t0, -1)
    print(" g  split0 emptyOK  loaded stored  arrive | mmaConvOK commit")
    for g in range(0, 60):
        print(f"{g:3d} {b[0][g]:7d} {b[1][g]:7d} {b[8][g]:7d} {b[9][g]:7d} {b[4][g]:7d} |"
              f" {b[2][g]:7d} {b[3][g]:7d}")
    print("half-0 unit j: slab wait start / done:", [(int(b[10][j]), int(b[11][j])) for j in range(0, 16, 2)])
    print("epilogue acc_full wake per unit:", b[5][:12].tolist(), "... last", b[5][b[5] >= 0].max())
    print("kernel entry", b[6][0], "exit", b[6][1], "(cycles, same origin)")
    ent, ex = buf[7][256:256 + 148], buf[7][:148]
    t0g = ent.min()
    print("globaltimer us: entry min/max", 0, (ent.max() - t0g) / 1e3, " exit min/median/max",
          (ex.min() - t0g) / 1e3, (np.median(ex) - t0g) / 1e3, (ex.max() - t0g) / 1e3)
    nkb = (Kd + 31) // 32
    d = np.diff(b[3][:200][b[3][:200] > 0])
    print("median cycles between MMA commits:", float(np.median(d)), "k-blocks per unit", nkb)


if __name__ == "__main__":
    main()
