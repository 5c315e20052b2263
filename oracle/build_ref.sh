#!/usr/bin/env bash
# Build the UNMODIFIED reference package (arxiv/paper_1205_1171, `hull3d`) into
# oracle/_ref/site so tests, smoke() and `bench.py --impl reference` can run the
# reference itself.  The reference's setup.py cythonizes src/hull3d/_ckernels.pyx
# and compiles it with `-O3 -ffp-contract=off` (pkg/setup.py:49-61).  The build
# writes into its source tree, so it runs from a throw-away copy under /tmp;
# the only output kept is oracle/_ref/ (git-ignored, NOT gpurun-ignored, so the
# prebuilt package travels to the GPU box, where /root/reference is absent).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${HULL3D_REFERENCE:-/root/reference/pkg}"
out="$here/_ref/site"
if [ ! -d "$src" ]; then
  echo "reference sources not found at $src; keeping prebuilt $out" >&2
  exit 0
fi
tmp="$(mktemp -d /tmp/h3dref.XXXXXX)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"
rm -rf "$out"
mkdir -p "$out"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$out" "$tmp/pkg"
python - "$out" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import hull3d, hull3d.kernels as K
assert K.has_compiled(), "reference compiled kernels failed to build"
print("reference built:", hull3d.__file__, "kernel =", K.active_name())
PY
