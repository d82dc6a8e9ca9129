for v in nostg stg nostg stg; do cp paper_2502_15734_b200/_lib_alt/$v.so paper_2502_15734_b200/_lib/libcc_b200.so; echo "== $v"; timeout 300 python tools/k1_ab.py 2>&1 | tail -2; done
