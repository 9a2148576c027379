# A/B of the feature backward variants and of stream overlap (config 3 frame, per-phase events)
run() { tag=$1; shift; env "$@" python bench.py --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > gpurun_out/r02f_$tag.log 2>&1; }
run base TK_FBWD_TMA=0
run tma1 TK_FBWD_CTAS=1
run tma2 TK_FBWD_CTAS=2
run tma3 TK_FBWD_CTAS=3
run tma4 TK_FBWD_CTAS=4
run ov_base TK_FBWD_TMA=0 TK_OVERLAP=1
run ov_tma1 TK_FBWD_CTAS=1 TK_OVERLAP=1
run ov_tma2 TK_FBWD_CTAS=2 TK_OVERLAP=1
python -m pytest tests -m gpu -x -q -k "c1c2 or fullsize" 2>&1 | tail -3
echo done
