#!/usr/bin/env bash
# Stage the UNMODIFIED reference package into oracle/_ref/ (git-ignored; gpurun ships it
# to the GPU box, where /root/reference does not exist).  Test infrastructure only:
# tests/test_gpu_level_a.py runs the reference's own run_serving_path with the B200
# scorer installed (plugin.install_into_zoserve), and bench.py's cpu_baseline times the
# reference's own lozo_step.  The product package never imports it.
#   usage: oracle/stage_ref.sh [/root/reference]
set -euo pipefail
SRC="${1:-/root/reference}/pkg/src/zoserve"
DST="$(cd "$(dirname "$0")" && pwd)/_ref"
if [ ! -d "$SRC" ]; then
  echo "stage_ref: $SRC not found (reference absent on this host); keeping $DST as is" >&2
  exit 0
fi
rm -rf "$DST/zoserve"
mkdir -p "$DST"
cp -r "$SRC" "$DST/zoserve"
find "$DST/zoserve" -name '__pycache__' -prune -exec rm -rf {} +
echo "staged $(ls "$DST/zoserve"/*.py | wc -l) reference modules into $DST/zoserve"
