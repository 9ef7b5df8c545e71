"""Pipeline timeline of the tensor-core gemm (CTA 0): per stage g, clock64
at TMA issue (after the empty wait), TMA landed (split warps' full wait),
split done, MMA issuer's conv wait done and commit.  Prints latencies."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200 import kernels as K
lib = K.lib()
M, N, Kd = [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1024x3072x4608").split("x")]
extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ldA, ldB = -(-Kd // 32) * 32, -(-N // 32) * 32
A = torch.rand(M, ldA, device="cuda") - 0.5
B = torch.rand(Kd, ldB, device="cuda") - 0.5
C = torch.zeros(M, ldB, device="cuda")
for flags in (extra, 16 | extra):
    lib.acct_tc_set_write_hi(flags)
    K.gemm_nn(M, N, Kd, 1.0, A.data_ptr(), ldA, B.data_ptr(), ldB, 0.0, C.data_ptr(), ldB, None, -1,
              K.GEMM_TC3XTF32, 0)
    torch.cuda.synchronize()
lib.acct_tc_set_write_hi(0)
tr = np.zeros((12, 512), dtype=np.int64)
assert lib.acct_tc_trace(tr.ctypes.data) == 0
n = int((tr[4] > 0).sum())
t0 = tr[0, 0]
tr = tr[:, :n] - t0
print(f"{M}x{N}x{Kd} flags={extra}: {n} stages traced; cycles per stage (steady) "
      f"{np.median(np.diff(tr[4][8:])):.0f}")
print("   g   issue  landed  split  mma_in  commit | tma_lat split_lat conv->mma  mma_dur")
for g in list(range(0, 12)) + list(range(n // 2, n // 2 + 8)):
    if g >= n:
        break
    i, l, c, m, e = tr[:5, g]
    print(f"{g:4d} {i:7d} {l:7d} {c:6d} {m:7d} {e:7d} | {l - i:7d} {c - l:9d} {m - c:9d} {e - m:8d}")
lat = tr[1] - tr[0]
if len(sys.argv) > 3:  # CTA-pair kernel: globaltimer ns; rows 5/6/7 = peer landed / split / relayed
    print("   g  lead: issue landed split mma_in commit | peer: landed split relayed   (ns)")
    for g in list(range(0, 10)) + list(range(n // 2, n // 2 + 6)):
        print(f"{g:4d} " + " ".join(f"{int(v):7d}" for v in tr[:8, g]))
    print(f"median ns: peer split {np.median(tr[6] - tr[5]):.0f}, relay after peer split "
          f"{np.median(tr[7] - tr[6]):.0f}, leader mma_in after relay {np.median(tr[3] - tr[7]):.0f}, "
          f"stage period {np.median(np.diff(tr[4][8:])):.0f}")
else:
    print(f"split parts: loads {np.median(tr[5] - tr[1]):.0f}  stores {np.median(tr[6] - tr[5]):.0f}  "
          f"fence {np.median(tr[7] - tr[6]):.0f}  arrive {np.median(tr[2] - tr[7]):.0f}")
print(f"median: tma {np.median(lat):.0f}  split {np.median(tr[2] - tr[1]):.0f}  "
      f"wait-for-mma {np.median(tr[3] - tr[2]):.0f}  mma-issue {np.median(tr[4] - tr[3]):.0f}")
