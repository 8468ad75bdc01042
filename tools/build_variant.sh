#!/bin/bash
# Build an A/B variant of libcfgsim.so with extra -D flags into
# paper_1707_02423_b200/variants/libcfgsim_<name>.so (git-ignored; travels to
# the GPU box).  Usage: tools/build_variant.sh <name> "-DFOO -DBAR"
set -e
name=$1; flags=$2
repo=$(cd "$(dirname "$0")/.." && pwd)
w=/tmp/cfgsim_variant_$name
rm -rf "$w"; mkdir -p "$w/pkg" "$w/include"
cp -r "$repo/paper_1707_02423_b200/csrc" "$w/pkg/csrc"; cp "$repo/include/"*.h "$w/include/"
rm -rf "$w/pkg/csrc/build"
make -s -j8 -C "$w/pkg/csrc" EXTRA="$flags" > "$w/make.log" 2>&1 || { tail -20 "$w/make.log"; exit 1; }
mkdir -p "$repo/paper_1707_02423_b200/variants"
cp "$w/pkg/libcfgsim.so" "$repo/paper_1707_02423_b200/variants/libcfgsim_$name.so"
echo "built variants/libcfgsim_$name.so ($flags)"
