#!/bin/bash
# A/B a kernel across alternative builds of libtri.so: tools/ab_lib.sh <lib>... -- <run_one args>
libs=(); while [ "$1" != "--" ]; do libs+=("$1"); shift; done; shift
cp paper_1609_01490_b200/libtri.so /tmp/libtri_orig.so
for l in "${libs[@]}"; do cp "$l" paper_1609_01490_b200/libtri.so; echo "== $l"; python tools/run_one.py "$@"; done
cp /tmp/libtri_orig.so paper_1609_01490_b200/libtri.so
