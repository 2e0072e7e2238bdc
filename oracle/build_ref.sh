#!/usr/bin/env bash
# Compiles the reference's own bookkeeping sources IN PLACE (read-only tree
# under /root/reference) plus oracle/ref_shim.cpp into oracle/_ref/.
# Nothing is copied into the repo.  workload.cpp needs nlohmann/json, which the
# reference does not vendor (proj/.gitignore:2); the image ships 3.11.3 inside
# cudnn_frontend, used read-only.  The reference's CMakeLists.txt is not used
# (it references missing subdirectories, CMakeLists.txt:14-16).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${SPECSIM_REFERENCE:-/root/reference}/proj"
JSON_DIR="$(python3 -c 'import sys,glob;p=glob.glob(sys.prefix+"/lib/python3*/site-packages/include/cudnn_frontend/thirdparty/nlohmann");print(p[0] if p else "")')"
if [ ! -d "$REF/src" ]; then echo "reference not present at $REF; skipping"; exit 0; fi
mkdir -p "$HERE/_ref"
SRCS="$REF/src/perf_model.cpp $HERE/ref_shim.cpp"
DEFS=""
if [ -n "$JSON_DIR" ] && [ -f "$JSON_DIR/json.hpp" ]; then
  SRCS="$SRCS $REF/src/workload.cpp"
else
  echo "nlohmann/json not found: building without workload.cpp" >&2
fi
g++ -std=c++20 -O2 -fPIC -shared -I"$REF/include" ${JSON_DIR:+-I"$JSON_DIR"} $SRCS -o "$HERE/_ref/libspecsim_ref.so"
echo "built $HERE/_ref/libspecsim_ref.so"
