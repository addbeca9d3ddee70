#!/bin/bash
# Build a kernel variant into paper_2605_20816_b200/lib/var/NAME.so:
#   bash tools/mkvar.sh NAME "-DPGX_EXP_FOO=1 ..."
set -e
cd "$(dirname "$0")/.."
mkdir -p paper_2605_20816_b200/lib/var
PGX_XFLAGS="$2" python -m paper_2605_20816_b200.build > /dev/null
cp paper_2605_20816_b200/lib/libpgx.so paper_2605_20816_b200/lib/var/$1.so
touch paper_2605_20816_b200/csrc/pgx_api.cu  # the next plain build recompiles
# NOTE: lib/libpgx.so now holds the VARIANT until that plain build runs
# (python -c "import __graft_entry__ as g; g.build()") -- rebuild before any gpurun of the product
echo "built $1 ($2)"
