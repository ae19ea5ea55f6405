#!/bin/bash
# Every sanitizer over the full small-case test list on the final build:
# memcheck / racecheck / synccheck on the pdg:: kernels, initcheck with every
# kernel instrumented (so torch's own writes count as initialisation).
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out/sanitizer
TOOLS="memcheck racecheck synccheck" SAN_TIMEOUT=500 bash tools/sanitize.sh
TOOLS=initcheck KNS= SAN_TIMEOUT=500 bash tools/sanitize.sh
echo all-done
