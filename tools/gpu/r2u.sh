#!/bin/bash
bash tools/gpu/gqa_ab.sh
bash tools/gpu/perf.sh r2u
