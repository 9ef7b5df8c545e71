"""Compare forced tensor-core tiles against an FP64 reference: max/normwise
error per tile for a few shapes, and where the error concentrates."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200 import kernels as K  # noqa: E402
lib = K.lib()
shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")]
tiles = [int(t) for t in sys.argv[2].split(",")]
for (M, N, Kd) in shapes:
    g = torch.Generator().manual_seed(5)
    A = torch.rand(M, Kd, generator=g) - 0.5
    B = torch.rand(Kd, N, generator=g) * 2 - 1
    ref = (A.double() @ B.double())
    ldA, ldB = -(-Kd // 32) * 32, -(-N // 32) * 32
    Ad = torch.zeros(M, ldA, device="cuda"); Ad[:, :Kd] = A.cuda()
    Bd = torch.zeros(Kd, ldB, device="cuda"); Bd[:, :N] = B.cuda()
    for t in tiles:
        lib.acct_tc_set_tile(t)
        Cd = torch.zeros(M, ldB, device="cuda")
        K.gemm_nn(M, N, Kd, 1.0, Ad.data_ptr(), ldA, Bd.data_ptr(), ldB, 0.0, Cd.data_ptr(), ldB,
                  None, -1, K.GEMM_TC3XTF32, 0)
        torch.cuda.synchronize()
        err = (Cd[:, :N].double().cpu() - ref).abs()
        scale = ref.abs().max().item()
        rows = err.max(dim=1).values
        cols = err.max(dim=0).values
        bad_r = (rows > 1e-5 * scale).nonzero().flatten().tolist()
        bad_c = (cols > 1e-5 * scale).nonzero().flatten().tolist()
        print(f"{M}x{N}x{Kd} tile {t}: max rel {err.max().item() / scale:.2e}  "
              f"bad rows {len(bad_r)} {bad_r[:6]}  bad cols {len(bad_c)} {bad_c[:6]}")
lib.acct_tc_set_tile(0)
