#!/bin/bash
for cfg in "32 8 1" "32 8 0" "16 8 1" "16 16 1"; do set -- $cfg; echo "WP=$1 CS=$2 LA=$3"; FEAST_WP=$1 FEAST_CS=$2 FEAST_LOOKAHEAD=$3 timeout 120 python tools/probe_c2.py C2 2>&1 | sed -n '1p;5,9p'; done
