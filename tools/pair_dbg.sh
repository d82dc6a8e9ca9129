# CTA-pair GEMM vs the 1-CTA plans at M=802 (and 5152 / 64)
echo "== pair forced"; CCB_SW_DEBUG=1 CCB_GEMM_FORCE=0,4 timeout 200 python tools/bench_gemm.py 802 2>&1 | cut -c1-110
echo "== pair dbg=1"; CCB_PAIR_DBG=1 CCB_GEMM_FORCE=0,4 timeout 200 python tools/bench_gemm.py 802 2>&1 | cut -c1-75
echo "== no pair (previous auto)"; CCB_GEMM_PAIR=0 timeout 200 python tools/bench_gemm.py 802 128 2048 2>&1 | cut -c1-75
echo "== auto"; timeout 200 python tools/bench_gemm.py 802 128 2048 2>&1 | cut -c1-75
