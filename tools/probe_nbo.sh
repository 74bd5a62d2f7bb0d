#!/bin/bash
for nbo in 64 128 256; do echo "NBO=$nbo"; FEAST_NBO=$nbo timeout 120 python tools/probe_c2.py C2 2>&1 | sed -n '1p;5,12p'; done
