#!/bin/bash
# Build libtri.so from a patched copy of the sources: tools/ab_variant.sh NAME PATCH.py
# PATCH.py runs with cwd = the copy's package dir (csrc/ inside); output: _ab/libtri_NAME.so
set -e
name=$1; patch=$(readlink -f "$2"); root=$(cd "$(dirname "$0")/.." && pwd)
w=/tmp/abv/$name; rm -rf "$w"; mkdir -p "$w"
cp -r "$root/include" "$w/"; mkdir -p "$w/paper_1609_01490_b200"
cp -r "$root/paper_1609_01490_b200/csrc" "$root/paper_1609_01490_b200/build.py" "$w/paper_1609_01490_b200/"
(cd "$w/paper_1609_01490_b200" && python "$patch" && python -c "import build; build.build()")
mkdir -p "$root/_ab"; cp "$w/paper_1609_01490_b200/libtri.so" "$root/_ab/libtri_$name.so"
echo "_ab/libtri_$name.so"
