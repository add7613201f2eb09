#!/usr/bin/env bash
# Regenerates the CWWF filter-data files (db2..db6, sym2..sym6) by running the
# reference's own offline generator, proj/tools/gen_wavelet_data.py (mpmath,
# 60 digits, deterministic), from a scratch copy: the generator writes to
# <tool>/../data and /root/reference is read-only.  The outputs are data, not
# source: they are committed under paper_2106_00554_b200/data/ because the
# product path needs the same taps and boundary matrices as the reference
# (SURVEY.md section 2 row 15, section 8c).
set -euo pipefail
REF=${REF:-/root/reference/proj}
OUT=${1:-$(cd "$(dirname "$0")/.." && pwd)/paper_2106_00554_b200/data}
TMP=$(mktemp -d /tmp/cwwgen.XXXXXX)
mkdir -p "$TMP/tools" "$OUT"
cp "$REF/tools/gen_wavelet_data.py" "$TMP/tools/"
python3 "$TMP/tools/gen_wavelet_data.py"
cp "$TMP"/data/*.cwwf "$OUT/"
md5sum "$OUT"/*.cwwf
rm -rf "$TMP"
