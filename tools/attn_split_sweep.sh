# ping-pong attention: key-split target / parts at config 2 and the 70B rank
for sp in "" "14,3" "11,4" "16,3" "10,4" "8,6" "12,4"; do
  echo "== split '$sp'"; CCB_ATTN_SPLIT=$sp timeout 300 python tools/attn_ab.py 4 20 2>&1 | grep -E "config2 r=.15|config2 r=.05|70B"
done
