#!/bin/bash
# Round-2 resume: verify HEAD (GPU suite, smoke, full N=1 bench + reference arm).
bash tools/gpu/check.sh r4a_check
bash tools/gpu/fullbench.sh r4a_full
