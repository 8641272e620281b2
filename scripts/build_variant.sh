#!/bin/bash
# Build an A/B variant of libvmap_b200.so with extra nvcc flags into scripts/bin/<name>/
# usage: scripts/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
name=$1; flags=$2
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/scripts/bin/$name
mkdir -p $out/obj
# objects listed in REBUILD (default: vm_kf32.o) are rebuilt with the flags,
# the others are reused from the main build
rebuild=${REBUILD:-vm_kf32.o}
for o in $root/paper_2302_01838_b200/_lib/obj/*.o; do
  case " $rebuild " in *" $(basename $o) "*) rm -f $out/obj/$(basename $o) ;; *) cp -p $o $out/obj/ ;; esac
done
make -s -C $root/paper_2302_01838_b200/csrc OUT=$out/libvmap_b200.so OBJDIR=$out/obj VMFLAGS="$flags" -j4 >/dev/null
echo $out/libvmap_b200.so
