#!/usr/bin/env bash
# experiment helper: run a command with an alternative libcjt_b200.so
set -e
ALT="$1"; shift
cp paper_1602_02618_b200/_lib/libcjt_b200.so /tmp/libcjt_orig.so
cp "$ALT" paper_1602_02618_b200/_lib/libcjt_b200.so
"$@" || true
cp /tmp/libcjt_orig.so paper_1602_02618_b200/_lib/libcjt_b200.so
