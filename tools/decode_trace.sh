run() {
  env "$@" timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 3 > gpurun_out/dec_x.json 2> gpurun_out/dec_x.err
  python -c "
import json
d=json.loads(open('gpurun_out/dec_x.json').read().strip().splitlines()[-1])['decode']
print('$*', d['ms_per_token'], d['roofline']['frac'], d['first_tokens'])
" || tail -3 gpurun_out/dec_x.err
}
cp paper_2502_15734_b200/_lib/libcc_b200.so /tmp/lib_s4.so
for st in 6 8; do cp tools/lib_s$st.so paper_2502_15734_b200/_lib/libcc_b200.so; echo "steps $st"; timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -k "qkv_matches or llama" 2>&1 | tail -1; done
for i in 1 2; do
  cp /tmp/lib_s4.so paper_2502_15734_b200/_lib/libcc_b200.so; run STEPS=4
  for st in 6 8; do cp tools/lib_s$st.so paper_2502_15734_b200/_lib/libcc_b200.so; run STEPS=$st; done
done
cp tools/lib_s6.so paper_2502_15734_b200/_lib/libcc_b200.so; echo "=== trace s6"; timeout 600 python tools/decode_trace.py 1 2>&1 | tail -4
cp /tmp/lib_s4.so paper_2502_15734_b200/_lib/libcc_b200.so
