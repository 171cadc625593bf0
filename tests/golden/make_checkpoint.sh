#!/usr/bin/env bash
# Regenerates tests/golden/ckpt_e64 with the reference's own ckpt::save
# (oracle/ckpt_tool.cpp, built by oracle/Makefile from /root/reference sources).
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
make -s -f "$ROOT/oracle/Makefile"
rm -rf "$ROOT/tests/golden/ckpt_e64"
"$ROOT/oracle/_ref/ckpt_tool" "$ROOT/tests/golden/ckpt_e64" 8
