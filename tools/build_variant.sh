#!/bin/bash
# Build an A/B variant of libsemb200.so with extra nvcc defines, reusing the main build's
# objects for every translation unit except the listed degree instantiations (default 7;
# 'sem3d' / 'krylov' name the other units):
#   tools/build_variant.sh NAME "-DFOO=1 -DBAR=2" [DEGREES...]  ->  build/var_NAME/libsemb200.so
# (run with SEM1D_LIB=build/var_NAME/libsemb200.so)
set -e
name=$1; flags=$2; shift 2
degs=${*:-7}
root=$(cd "$(dirname "$0")/.." && pwd)
obj=$root/build/var_$name/obj
mkdir -p "$obj"
cp -p "$root"/build/obj/*.o "$obj"/
for d in $degs; do
  case $d in
    sem3d|krylov) rm -f "$obj/$d.o" ;;          # other translation units by name
    *) rm -f "$obj/inst_$d.o" ;;
  esac
done
rm -f "$obj/capi.o"
make -s -C "$root/paper_1806_01422_b200/csrc" OBJDIR="$obj" LIB="$root/build/var_$name/libsemb200.so" \
     EXTRA_NVFLAGS="$flags" -j8
rm -rf "$obj"
echo "built build/var_$name/libsemb200.so"
