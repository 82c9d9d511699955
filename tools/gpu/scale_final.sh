#!/bin/bash
bash tools/gpu/scale.sh scale_final 4 ""
bash tools/gpu/scale.sh scale_final 2 ""
