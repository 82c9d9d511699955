#!/bin/bash
bash tools/gpu/gqa_ab.sh
bash tools/gpu/tables_dense.sh
