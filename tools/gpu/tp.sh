#!/bin/bash
C3K=5 PLANTED=1 PAIRS=1 timeout 300 python tools/trace_dkv.py 2>&1 | grep -v Warn | tail -16
