"""Time acct_conv3x3_tc_f32 at the yolov2-tiny layer shapes (16 images,
column-interleaved batch), optionally with ACCT_CONV_DBG set to skip the
operand build (1), the MMAs (2) or the epilogue (4) -- pipeline analysis.

    python tools/conv_probe.py            # prints us per image per layer
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_1811_03882_b200 import kernels as K  # noqa: E402


def main():
    P = 16
    for (c, h, w, M) in ((16, 208, 208, 32), (32, 104, 104, 64), (64, 52, 52, 128)):
        N, Kd = h * w, 9 * c
        ld = -(-N // 32) * 32
        lda = -(-Kd // 32) * 32
        im = torch.randn((c, P * ld), device="cuda")
        A = torch.randn((M, lda), device="cuda")
        col = torch.zeros((Kd, P * ld), device="cuda")
        C = torch.zeros((M, P * ld), device="cuda")
        bias = torch.randn(M, device="cuda")
        s = torch.cuda.current_stream().cuda_stream
        P2 = (h // 2) * (w // 2)
        ldp = -(-P2 // 32) * 32
        pool = torch.zeros((M, P * ldp), device="cuda")
        pidx = torch.zeros((M, P * ldp), dtype=torch.int32, device="cuda")
        pl = ((pool.data_ptr(), P * ldp, ldp, pidx.data_ptr(), P * ldp, ldp, P - 1)
              if os.environ.get("POOL") == "1" else None)

        def run():
            K.conv3x3_tc(im.data_ptr(), P * ld, ld, c, h, w, col.data_ptr(), P * ld, ld, M,
                         A.data_ptr(), lda, 0.0, C.data_ptr(), P * ld, ld, bias.data_ptr(),
                         K.ACT_LEAKY, P, s, col_from=P - 1, pool=pl)
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            run()
        e1.record()
        e1.synchronize()
        print(f"c{c} {h}x{w} M{M}: {e0.elapsed_time(e1) / 20 / P * 1e3:.2f} us/img")


if __name__ == "__main__":
    main()
