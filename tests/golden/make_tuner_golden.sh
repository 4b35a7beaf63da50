#!/usr/bin/env bash
# Regenerates tests/golden/tuner/ from the reference sources (needs
# /root/reference and oracle/_ref/libwgtune_ref.a from oracle/build_ref.sh).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/../.." && pwd)"
JSON_INC=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
bash "$ROOT/oracle/build_ref.sh" > /dev/null
g++ -std=c++20 -O2 -I/root/reference/proj/include -I"$JSON_INC" "$ROOT/tests/golden/make_tuner_golden.cpp" \
  "$ROOT/oracle/_ref/libwgtune_ref.a" -pthread -o /tmp/make_tuner_golden
rm -rf "$ROOT/tests/golden/tuner"
/tmp/make_tuner_golden "$ROOT/tests/golden/tuner"
