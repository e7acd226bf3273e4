# Config 5 with the committed wisdom as anchors and non-cubic / in-between query shapes.
OUT=${OUT:-gpurun_out/port2}
mkdir -p $OUT
timeout 5000 python -m paper_2303_12374_b200.portability --anchor-wisdom wisdom --evals 40 \
  --queries 300,384,640x640x320,1024x512x256,768x768x192 --out $OUT/portability.json > $OUT/log.txt 2>&1
echo rc=$?; grep -E "selected|ppm" $OUT/log.txt | tail -30
