"""Does tcgen05 kind::tf32 truncate FP32 operands (ignore the low 13 bits)?
Runs the tensor-core gemm with explicit hi (masked) operands and with raw
FP32 in place of hi; identical bits => the MMA truncates."""
import sys, ctypes as C
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200 import kernels as K
lib = K.lib()
lib.acct_tc_set_write_hi.argtypes = [C.c_int]
for (M, N, Kd) in [(128, 128, 64), (1024, 169, 4608), (16, 4096, 27), (256, 676, 1152)]:
    g = torch.Generator().manual_seed(1)
    A = (torch.rand(M, Kd, generator=g) - 0.5).cuda(); B = (torch.rand(Kd, N, generator=g) * 2 - 1).cuda()
    ldA, ldB = -(-Kd // 32) * 32, -(-N // 32) * 32
    Ad = torch.zeros(M, ldA, device="cuda"); Ad[:, :Kd] = A
    Bd = torch.zeros(Kd, ldB, device="cuda"); Bd[:, :N] = B
    outs = []
    for wh in (1, 0):
        lib.acct_tc_set_write_hi(wh)
        Cd = torch.zeros(M, ldB, device="cuda")
        K.gemm_nn(M, N, Kd, 1.0, Ad.data_ptr(), ldA, Bd.data_ptr(), ldB, 0.0, Cd.data_ptr(), ldB, None, -1, K.GEMM_TC3XTF32, 0)
        torch.cuda.synchronize()
        outs.append(Cd[:, :N].clone())
    ref = (A.double() @ B.double())
    same = torch.equal(outs[0], outs[1])
    e = [float(((o.double() - ref).abs().max() / ref.abs().max())) for o in outs]
    print(f"{M}x{N}x{Kd}: bit-identical={same} maxrel(hi)={e[0]:.2e} maxrel(raw)={e[1]:.2e} ndiff={int((outs[0]!=outs[1]).sum())}")
lib.acct_tc_set_write_hi(1)
