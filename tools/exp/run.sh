#!/bin/bash
# Swap library variants and run the attention probe (development experiments).
cd "$(dirname "$0")/../.."
cp paper_2602_16249_b200/libaffmae_b200.so /tmp/keep.so
for v in "$@"; do
  cp tools/exp/lib_$v.so paper_2602_16249_b200/libaffmae_b200.so
  echo "== $v"; timeout 120 python tools/probe_attn.py 32 2>&1 | tail -2
done
cp /tmp/keep.so paper_2602_16249_b200/libaffmae_b200.so
