#!/bin/sh
# Stage the unmodified reference package (gridcast) into baseline/_ref (git-ignored; travels to the GPU box with
# gpurun) so the integration tests can import it where /root/reference does not exist.  Offline install from the
# image's wheelhouse; the build writes into its source tree, so it runs from a copy under /tmp.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/gridcast_src && cp -r /root/reference/pkg /tmp/gridcast_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade /tmp/gridcast_src
