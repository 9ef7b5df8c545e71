"""Device time of one gemm_nn launch (captured 20x in a CUDA graph, so no
host overhead), per shape and per debug knob of the tensor-core kernel:
  flags bit1 = skip hi/lo split, bit2 = skip MMAs, bit3 = skip epilogue."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200 import kernels as K
lib = K.lib()
SHAPES = [(16, 173056, 27), (32, 43264, 144), (64, 10816, 288), (128, 2704, 576), (256, 676, 1152),
          (512, 169, 2304), (1024, 169, 4608), (512, 169, 9216), (425, 169, 512), (4096, 4096, 4096)]
flag_sets = [int(f) for f in sys.argv[1].split(",")] if len(sys.argv) > 1 else [0]
if len(sys.argv) > 2:   # "MxNxK,MxNxK,..."
    SHAPES = [tuple(int(v) for v in t.split("x")) for t in sys.argv[2].split(",")]
modes = {"tc": K.GEMM_TC3XTF32, "simt": K.GEMM_SIMT, "auto": K.GEMM_AUTO}
for (M, N, Kd) in SHAPES:
    ldA, ldB = -(-Kd // 32) * 32, -(-N // 32) * 32
    A = torch.rand(M, ldA, device="cuda") - 0.5
    B = torch.rand(Kd, ldB, device="cuda") - 0.5
    C = torch.zeros(M, ldB, device="cuda")
    line = f"{M:5d}x{N:6d}x{Kd:5d}:"
    for name, mode in modes.items():
        for fl in (flag_sets if name == "tc" else [0]):
            lib.acct_tc_set_write_hi(fl)
            s = torch.cuda.Stream()
            reps = 20 if M * N * Kd < 1e10 else 4
            with torch.cuda.stream(s):
                K.gemm_nn(M, N, Kd, 1.0, A.data_ptr(), ldA, B.data_ptr(), ldB, 0.0, C.data_ptr(), ldB, None, -1, mode, s.cuda_stream)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(reps):
                        K.gemm_nn(M, N, Kd, 1.0, A.data_ptr(), ldA, B.data_ptr(), ldB, 0.0, C.data_ptr(), ldB, None, -1, mode, s.cuda_stream)
            g.replay(); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            line += f"  {name}{fl if name == 'tc' else ''}={us:7.1f}us"
    lib.acct_tc_set_write_hi(0)
    print(line + f"   ({2*M*N*Kd/1e9:.2f} GF)", flush=True)
