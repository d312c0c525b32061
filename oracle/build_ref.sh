#!/usr/bin/env bash
# Compile the reference's own execution core (one Cython source) from where it
# lies under /root/reference into oracle/_ref/.  Nothing from the reference is
# copied into the repository: the .pyx is cythonized in a /tmp scratch dir and
# only the resulting shared object lands in oracle/_ref/ (git-ignored, but it
# travels to the GPU box with the snapshot).  Uses /usr/bin/gcc because the
# image's default CC (/opt/gcc) cannot link -fopenmp (no libgomp.spec).
set -euo pipefail
REF=${REFERENCE_ROOT:-/root/reference}
SRC="$REF/pkg/src/vecchiagp/engine/_kernels.pyx"
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
    echo "build_ref: $SRC not present (GPU box?) - keeping any prebuilt oracle/_ref" >&2
    exit 0
fi
TMP="$(mktemp -d /tmp/vgp_ref_XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp "$SRC" "$TMP/_kernels.pyx"
PY=${PYTHON:-python}
( cd "$TMP" && "$PY" -m cython -3 -X boundscheck=False -X wraparound=False \
      -X cdivision=True -X initializedcheck=False _kernels.pyx -o _kernels.c )
INC_PY="$("$PY" -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
INC_NP="$("$PY" -c 'import numpy; print(numpy.get_include())')"
EXT="$("$PY" -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
mkdir -p "$OUT"
/usr/bin/gcc -O3 -fopenmp -ffp-contract=off -fPIC -shared -fwrapv \
    -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -I"$INC_PY" -I"$INC_NP" "$TMP/_kernels.c" -o "$OUT/_kernels$EXT" -lm
echo "build_ref: wrote $OUT/_kernels$EXT"
