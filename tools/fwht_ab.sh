#!/bin/bash
for mb in 16 8 24 32; do echo "== chunk $mb"; MCK_FWHT_CHUNK_MB=$mb timeout 120 python tools/sweep_fwht.py 14; done
