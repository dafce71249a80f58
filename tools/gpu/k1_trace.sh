for cfg in "STAR_K1_SEQ=0" "STAR_K1_SEQ=1" "STAR_K1_SEQ=1 STAR_K1_POLY=1"; do env $cfg timeout 300 python tools/k1_trace.py; done
