run() {
  env "$@" timeout 900 python bench.py --no-baselines --no-cpu --tiers 0 --steps 3 > gpurun_out/dec_x.json 2> gpurun_out/dec_x.err
  python -c "
import json
d=json.loads(open('gpurun_out/dec_x.json').read().strip().splitlines()[-1])['decode']
print('$*', d['ms_per_token'], d['roofline']['frac'], d['first_tokens'])
" || tail -3 gpurun_out/dec_x.err
}
cp paper_2502_15734_b200/_lib/libcc_b200.so /tmp/lib_base.so
for i in 1 2; do
  cp /tmp/lib_base.so paper_2502_15734_b200/_lib/libcc_b200.so; run ATTN_LB=3; run ATTN_LB=3 CCB_DT_STAGE_PRE=2; run ATTN_LB=3 CCB_DT_STAGE_PRE=0
  cp tools/lib_a2.so paper_2502_15734_b200/_lib/libcc_b200.so; run ATTN_LB=2
done
cp /tmp/lib_base.so paper_2502_15734_b200/_lib/libcc_b200.so
