#!/bin/bash
for wp in 16 32 64; do echo "WP=$wp"; FEAST_WP=$wp timeout 120 python tools/probe_c2.py C2 2>&1 | sed -n '1p;5,9p'; done
