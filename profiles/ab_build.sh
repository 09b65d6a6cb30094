#!/bin/bash
# Build the committed HEAD's library as profiles/libgr4ad_base.so (A/B runs:
# GR4AD_LIB=profiles/libgr4ad_base.so selects it) without touching the tree.
set -e
W=$(mktemp -d)
git -C "$(dirname "$0")/.." archive HEAD paper_2602_22732_b200/csrc include | tar -x -C "$W"
make -C "$W/paper_2602_22732_b200/csrc" -j8 BUILD=build_base LIB="$(cd "$(dirname "$0")"; pwd)/libgr4ad_base.so" > /dev/null
rm -rf "$W"
