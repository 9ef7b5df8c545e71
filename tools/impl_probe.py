"""yolov2-tiny L13 (1024 ch 13x13 -> 512, 16 images) through the implicit-im2col
pair gemm, 4 launches (for ncu: skip 3, capture 1)."""
import os
import sys
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
from paper_1811_03882_b200 import kernels as K  # noqa: E402

c, h, w, M, P = 1024, 13, 13, 512, 16
HW, Kd, ld = h * w, 9 * c, 172
im = torch.rand(c, P * ld, device="cuda")
A = torch.rand(M, Kd, device="cuda")
col = torch.zeros(Kd, P * ld, device="cuda")
C = torch.zeros(M, P * ld, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    K.conv3x3_gemm_tc(im.data_ptr(), P * ld, ld, c, h, w, col.data_ptr(), P * ld, ld, M,
                      A.data_ptr(), Kd, 0.0, C.data_ptr(), P * ld, ld, None, K.ACT_LEAKY, P, s,
                      col_from=P - 1)
torch.cuda.synchronize()
