#!/bin/bash
LLMP_PART=2 bash tools/prof_kernel.sh pa2 "k_part" 7 40 42 2 5
rm -f gpurun_out/pa2_raw.csv
