#!/bin/bash
# Build an A/B variant of the library with extra nvcc defines (diagnostic):
#   bash scripts/build_variant.sh librecmg_a.so -DRECMG_ROW_L2_AHEAD=0
OUT=$1; shift
cd "$(dirname "$0")/../paper_2511_08568_b200/csrc" && \
make -s -j8 OBJDIR=../../build/variant_${OUT%.so} OUT=../${OUT} EXTRA="$*"
