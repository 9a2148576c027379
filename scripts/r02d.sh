#!/bin/bash
# round 2d: HBM stream ceilings, records-per-Gaussian distribution, kLongSeg A/B (config 3 frame)
mkdir -p gpurun_out
./scripts/bw_probe > gpurun_out/r02d_bw.txt 2>&1
python scripts/seg_hist.py > gpurun_out/r02d_seg.txt 2>&1
python scripts/seg_hist.py 100000 640 480 16 >> gpurun_out/r02d_seg.txt 2>&1
bash scripts/ab_libs.sh "k_feat_bwd|k_gather_staged" "--steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" \
  default ls128 ls256 ls512 > gpurun_out/r02d_ab.txt 2>&1
bash scripts/ab_libs.sh "k_feat_bwd" "--config c1 --k 16 --steps 10 --warmup 3 --no-e2e --no-mapping --no-extras --no-cpu" \
  default ls128 ls256 >> gpurun_out/r02d_ab.txt 2>&1
cat gpurun_out/r02d_bw.txt gpurun_out/r02d_seg.txt gpurun_out/r02d_ab.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; python -c "import json;d=json.loads(open(\"gpurun_out/r02d_bench.json\").read().strip().splitlines()[-1]);print(d[\"value\"], json.dumps(d[\"extras\"][\"mapedit\"]))"
