"""Quick tensor-core gemm check/timing (dev tool)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
from paper_1811_03882_b200 import kernels as K
shapes = [(128,128,32),(128,128,64),(256,256,256),(64,10816,288),(128,2704,576),(256,676,1152),(512,169,2304),(1024,169,4608),(512,169,9216),(425,169,512),(130,129,33),(200,300,64),(4096,4096,4096)]
for M,N,Kd in shapes:
    g = torch.Generator().manual_seed(0)
    A = torch.rand(M,Kd,generator=g)-0.5; B = torch.rand(Kd,N,generator=g)*2-1
    ldA = -(-Kd//32)*32; ldB = -(-N//32)*32
    Ad = torch.zeros(M,ldA,device='cuda'); Ad[:,:Kd]=A.cuda()
    Bd = torch.zeros(Kd,ldB,device='cuda'); Bd[:,:N]=B.cuda()
    Cd = torch.zeros(M,ldB,device='cuda')
    ref = (A.double()@B.double()).float()
    s = torch.cuda.current_stream().cuda_stream
    for mode in (K.GEMM_TC3XTF32, K.GEMM_SIMT):
        Cd.zero_()
        try:
            K.gemm_nn(M,N,Kd,1.0,Ad.data_ptr(),ldA,Bd.data_ptr(),ldB,0.0,Cd.data_ptr(),ldB,None,-1,mode,s)
            torch.cuda.synchronize()
        except Exception as e:
            print(M,N,Kd,mode,"ERR",e); continue
        got = Cd[:,:N].cpu()
        err = float((got-ref).abs().max()/ref.abs().max())
        nerr = float((got-ref).double().norm()/ref.double().norm())
        # timing
        reps = 20 if M*N*Kd < 1e10 else 5
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            K.gemm_nn(M,N,Kd,1.0,Ad.data_ptr(),ldA,Bd.data_ptr(),ldB,0.0,Cd.data_ptr(),ldB,None,-1,mode,s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)/reps
        print(f"{M:5d} {N:6d} {Kd:5d} mode={mode} maxrel={err:.2e} normrel={nerr:.2e} {ms*1e3:9.1f}us {2*M*N*Kd/ms/1e9:8.2f} TFLOP/s", flush=True)
