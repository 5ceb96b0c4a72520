#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Compiles the reference's lattice-core from its
# sources where they lie under /root/reference (never copied) plus our C shim
# into oracle/_ref/libref_lattice.so. The reference includes <json.hpp>
# from its (absent, git-ignored) vendor/ dir; nlohmann json 3.11.3 from the
# image stands in for it. Exits 0 without building when /root/reference is
# absent (GPU boxes use the prebuilt fixtures in tests/golden/).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
ref=/root/reference/proj/src/core
json_dir=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
if [ ! -f "$ref/lattice.cpp" ] || [ ! -f "$json_dir/json.hpp" ]; then
  echo "build_ref.sh: reference or json.hpp not present; skipping" >&2
  exit 0
fi
mkdir -p "$here/_ref"
g++ -std=c++20 -O2 -fPIC -shared -I"$ref" -I"$json_dir" \
    "$ref/lattice.cpp" "$here/ref_lattice_shim.cpp" -o "$here/_ref/libref_lattice.so"
echo "built $here/_ref/libref_lattice.so"
