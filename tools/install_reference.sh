#!/bin/bash
# Install the UNMODIFIED reference package (ale_minihydro, pure Python) into baseline/_ref
# for bench.py's reference arm and cpu_baseline.  /root/reference is read-only and the
# setuptools build writes into its source tree, so it builds from a copy under /tmp.
# baseline/_ref is git-ignored but travels to the GPU box with the gpurun snapshot.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC: keeping the existing baseline/_ref" >&2; exit 0; }
TMP="$(mktemp -d /tmp/refpkg.XXXXXX)"
cp -r "$SRC/." "$TMP/"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP" >/dev/null
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import ale_minihydro.hydro; print('reference installed:', ale_minihydro.__file__)"
