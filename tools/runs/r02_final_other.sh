# the other configs' lines with the final bench.py (dataset-cycling baseline + weights-at-init twin)
for c in c1 c2 c3 c5; do
  timeout 1500 python bench.py --config $c > gpurun_out/fo_$c.json 2> gpurun_out/fo_$c.err; echo "$c rc=$?"
done
