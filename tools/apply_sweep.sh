#!/usr/bin/env bash
# Standalone-MVM schedule sweep (run under gpurun from the repo root):
# near GEMV kernel variants x coupling placement, y compared across variants.
out=gpurun_out/${1:-sweep}
shift
mkdir -p $out
run() {  # tag env...
  local tag=$1; shift
  env "$@" timeout 600 python tools/apply_probe.py --save $out/y_$tag.npy $PROBE_ARGS > $out/$tag.json 2> $out/$tag.err
  echo "$tag $(cat $out/$tag.json | tail -1)"
}
run old ${BASE_ENV:-PHM_NEAR_GEMV=0}
while [ $# -gt 0 ]; do
  tag=$1; shift; envs=$1; shift
  run $tag $envs
done
python - $out <<'PY'
import sys, numpy as np, glob, os
d = sys.argv[1]
ref = np.load(f"{d}/y_old.npy")
for f in sorted(glob.glob(f"{d}/y_*.npy")):
    y = np.load(f)
    print(os.path.basename(f), np.linalg.norm(y - ref) / np.linalg.norm(ref))
PY
