import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_1811_03882_b200 import kernels as K
P, (c, h, w, M) = 16, (16, 208, 208, 32)
N, Kd = h*w, 9*c
ld, lda = -(-N//32)*32, -(-Kd//32)*32
im = torch.randn((c, P*ld), device="cuda"); A = torch.randn((M, lda), device="cuda")
col = torch.zeros((Kd, P*ld), device="cuda"); C = torch.zeros((M, P*ld), device="cuda")
bias = torch.randn(M, device="cuda")
P2 = (h//2)*(w//2); ldp = -(-P2//32)*32
pool = torch.zeros((M, P*ldp), device="cuda"); pidx = torch.zeros((M, P*ldp), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(4):
    K.conv3x3_tc(im.data_ptr(), P*ld, ld, c, h, w, col.data_ptr(), P*ld, ld, M, A.data_ptr(), lda, 0.0, C.data_ptr(), P*ld, ld, bias.data_ptr(), K.ACT_LEAKY, P, s, col_from=P-1, pool=(pool.data_ptr(), P*ldp, ldp, pidx.data_ptr(), P*ldp, ldp, P-1))
torch.cuda.synchronize()
