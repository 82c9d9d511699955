#!/bin/bash
bash tools/gpu/dbg_hang.sh
bash tools/gpu/ab_epi.sh
