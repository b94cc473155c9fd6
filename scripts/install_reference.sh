# Offline install of the unmodified reference (densefeed + its bindings) into baseline/_ref (git-ignored, travels
# with gpurun).  The build writes into its source tree, so it installs from a copy under /tmp.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/refcopy && cp -r /root/reference /tmp/refcopy
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" /tmp/refcopy/pkg /tmp/refcopy/pkg/bindings
