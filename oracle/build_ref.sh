#!/bin/sh
# ORACLE — TEST INFRASTRUCTURE ONLY. Compiles oracle/ref_kat.cpp against the
# reference headers where they lie (read-only, never copied) into oracle/_ref/.
set -e
REF=${REF:-/root/reference}
HERE=$(cd "$(dirname "$0")" && pwd)
mkdir -p "$HERE/_ref"
g++ -std=c++20 -O2 -I"$REF/proj/include" "$HERE/ref_kat.cpp" -o "$HERE/_ref/ref_kat"
