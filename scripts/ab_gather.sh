# A/B of the feature gather variants (config 3 frame, per-phase events) + parity of the gathers
run() { tag=$1; shift; env "$@" python bench.py --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu > gpurun_out/r02g_$tag.log 2>&1; }
python -m pytest tests -m gpu -x -q -k "feature or fused or parity or c1c2 or fullsize_feature or mapping" 2>&1 | tail -2
run staged TK_GATHER_PIPE=0
run pipe224 TK_GATHER_PIPE_KB=224
run pipe112 TK_GATHER_PIPE_KB=112
run pipe160 TK_GATHER_PIPE_KB=160
run pipe72 TK_GATHER_PIPE_KB=72
echo done
