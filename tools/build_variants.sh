#!/bin/bash
# Build tuning variants of the library into tools/variants/<name>/ (git-ignored).
set -e
cd "$(dirname "$0")/.."
build() {
  name=$1; shift
  make -s BUILD=build/var_$name LIBDIR=tools/variants/$name XFLAGS="$*" tools/variants/$name/libglare_b200.so >/dev/null
  grep -A2 "cross_filter_kernelILb1E" tools/variants/$name/ptxas.log | grep -oE "Used [0-9]+ registers|[0-9]+ bytes spill stores" | tr '\n' ' '; echo " <- $name"
}
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  build "$name" $flags &
done
wait
