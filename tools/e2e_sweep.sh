#!/bin/bash
# end-to-end leg vs number of upload chunks, and the per-rank work of strong scaling measured on one GPU
for c in 8 12 16 24 32; do
  VB200_UPLOAD_CHUNKS=$c python bench.py --steps 20 --warmup 3 --no-extras --no-cpu-baseline > /tmp/b_$c.json 2>/dev/null
  python - <<PY
import json; d=json.load(open("/tmp/b_$c.json")); print("chunks", $c, "e2e ms mean", round(d["e2e"]["ms_per_step"],3), "min", d["e2e"]["ms_min"])
PY
done
for n in 131072 262144 524288 1048576; do
  python bench.py --n $n --steps 30 --warmup 5 --no-extras --no-cpu-baseline > /tmp/n_$n.json 2>/dev/null
  python - <<PY
import json; d=json.load(open("/tmp/n_$n.json")); print("n", d["config"]["n_total"], "ms_per_step", round(d["ms_per_step"],4), "kernel_ms", round(d["roofline"]["kernel_ms"],4), "obs/s", round(d["value"]/1e6,1), "M", d["config"]["l2_policy"][:24])
PY
done
