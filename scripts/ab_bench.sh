#!/bin/bash
# A/B timing of builds of libsk_b200.so on the same box, interleaved:
#   bash scripts/ab_bench.sh <tag> <reps> "<lib1> <lib2> ..." <bench args...>
# lib = a path to a libsk_b200.so (scripts/build_variant.py), "tree" for the in-tree build, or
# "tree:VAR=value" for the in-tree build with an environment variable set.
set -u
tag=$1; reps=$2; libs=$3; shift 3
for i in $(seq 1 $reps); do
  k=0
  for l in $libs; do
    k=$((k + 1))
    if [ "$l" = tree ]; then
      python bench.py "$@" > gpurun_out/ab_${tag}_${k}_$i.json 2>/dev/null
    elif [ "${l%%:*}" = tree ]; then  # tree:VAR=value -- the in-tree build with an environment setting
      env "${l#tree:}" python bench.py "$@" > gpurun_out/ab_${tag}_${k}_$i.json 2>/dev/null
    else
      SK_B200_LIB=$PWD/$l python bench.py "$@" > gpurun_out/ab_${tag}_${k}_$i.json 2>/dev/null
    fi
  done
done
python - "$tag" "$reps" $libs <<'PY'
import json, sys
tag, reps, libs = sys.argv[1], int(sys.argv[2]), sys.argv[3:]
for k, l in enumerate(libs, 1):
    ms = []
    for i in range(1, reps + 1):
        try:
            d = json.loads(open(f"gpurun_out/ab_{tag}_{k}_{i}.json").read().strip().splitlines()[-1])
            ms.append(d["ms_per_step"])
        except Exception:
            ms.append(float("nan"))
    print(tag, l, " ".join(f"{x:.4f}" for x in ms), "mean %.4f" % (sum(ms) / len(ms)))
PY
