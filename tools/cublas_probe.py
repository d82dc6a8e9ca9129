import torch
for (N,K) in ((6144,4096),(4096,4096),(28672,4096),(4096,14336)):
    A=torch.randn((802,K),device='cuda').bfloat16(); B=(torch.randn((N,K),device='cuda')/64).bfloat16()
    for _ in range(3): C=torch.matmul(A,B.T)
torch.cuda.synchronize()
