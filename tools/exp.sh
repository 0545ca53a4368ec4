#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
timeout 120 ./build/umma_bench > $OUT/umma_bench.txt 2>&1
echo done > $OUT/DONE
