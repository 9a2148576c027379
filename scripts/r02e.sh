#!/bin/bash
# round 2e: band-major long-segment feature backward: parity + A/B (config 1 K = 16 / 8, config 3)
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q -k "long or c1c2 or fullsize or stress or mapping or lazy" > gpurun_out/r02e_tests.txt 2>&1
tail -3 gpurun_out/r02e_tests.txt
for v in default ls256 ls256i64; do
  [ $v = default ] && unset TK_RENDER_LIB || export TK_RENDER_LIB=$PWD/paper_2602_06991_b200/lib/$v/libtkrender.so
  [ $v = default ] || TK_RENDER_LIB=$TK_RENDER_LIB python -m pytest tests -m gpu -x -q -k "long or c1c2" > gpurun_out/r02e_tests_$v.txt 2>&1
  echo "$v tests: $(tail -1 gpurun_out/r02e_tests_$v.txt 2>/dev/null)"
done
unset TK_RENDER_LIB
bash scripts/ab_libs.sh "k_feat_bwd|k_long|k_gather_staged" "--config c1 --k 16 --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" \
  default ls256 ls256i64 > gpurun_out/r02e_ab.txt 2>&1
bash scripts/ab_libs.sh "k_feat_bwd|k_long" "--config c1 --k 8 --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" \
  default ls256 >> gpurun_out/r02e_ab.txt 2>&1
bash scripts/ab_libs.sh "k_feat_bwd|k_long" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" \
  default ls256 >> gpurun_out/r02e_ab.txt 2>&1
cat gpurun_out/r02e_ab.txt
PYTHONPATH=. python scripts/seg_hist.py > gpurun_out/r02e_seg.txt 2>&1
PYTHONPATH=. python scripts/seg_hist.py 100000 640 480 16 >> gpurun_out/r02e_seg.txt 2>&1
cat gpurun_out/r02e_seg.txt
