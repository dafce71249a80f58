# K2q split fold with grouped loads (EG = 4) vs the baseline library: query encode timings
# (l_q = 8, 32 at 16K / 128K rows), alternating.  Needs paper_2411_17116_b200/libstar_attn_base.so.
for i in 1 2 3; do
  echo "== base"; STAR_LIB_PATH=paper_2411_17116_b200/libstar_attn_base.so QB_LQ=8,32 timeout 120 python tools/query_bench.py
  echo "== new"; QB_LQ=8,32 timeout 120 python tools/query_bench.py
done
for i in 1 2; do
  echo "== base decode"; STAR_LIB_PATH=paper_2411_17116_b200/libstar_attn_base.so timeout 120 python tools/k2_overhead.py 4096 16384 131072
  echo "== new decode"; timeout 120 python tools/k2_overhead.py 4096 16384 131072
done
