#!/bin/sh
# Stage the reference package's own unit tests (read-only /root/reference) into
# baseline/_ref/tests -- git-ignored, NOT gpurun-ignored -- so they travel to
# the GPU box and tests/test_reference_suite.py runs them against the `cfcent`
# import shim (the B200 package).  Nothing of the reference enters git history.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg/tests}
mkdir -p "$ROOT/baseline/_ref/tests"
cp "$SRC"/*.py "$ROOT/baseline/_ref/tests/"
printf '[pytest]\naddopts = -p no:cacheprovider\n' > "$ROOT/baseline/_ref/tests/pytest.ini"
ls "$ROOT/baseline/_ref/tests"
