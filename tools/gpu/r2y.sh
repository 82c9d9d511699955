#!/bin/bash
bash tools/gpu/balance_final.sh 4 8 balance_final3
