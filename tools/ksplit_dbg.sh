cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2502_15734_b200 import _native as N
M, Nn, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A = torch.randn((M, K), device='cuda').bfloat16(); B = (torch.randn((Nn, K), device='cuda') / 64).bfloat16()
C = torch.zeros((M, Nn), device='cuda')
f = lambda: N.call('cc_gemm', N.ptr(A), K, N.ptr(B), K, N.ptr(C), Nn, M, Nn, K, N.EPI_RESID_ADD, N.BF16, 1, N.stream_ptr())
for _ in range(3): f()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): f()
b.record(); torch.cuda.synchronize()
print(sys.argv[1:], 'us', round(a.elapsed_time(b) / 20 * 1e3, 1))
PY
for f in "0,4" "2,5" "3,5"; do for d in 0 16 32 1; do echo "force=$f dbg=$d"; CCB_GEMM_FORCE=$f CCB_PAIR_DBG=$d timeout 120 python /tmp/one.py 290 4096 4096; CCB_GEMM_FORCE=$f CCB_PAIR_DBG=$d timeout 120 python /tmp/one.py 290 4096 14336; done; done 2>&1 | grep -v Warn
