#!/bin/bash
# Native (C-ABI, no Python) step times across the BASELINE configs.
B=paper_2506_01969_b200/lib/etap_bench
$B --batch 1 --ctx 1024 --heads 16 --iters 500 --graph 50
for c in 1024 2048 4096 8192 16384 32768 65536; do $B --batch 16 --ctx $c --heads 16 --iters 300 --graph 30; done
$B --batch 16 --ctx 65536 --heads 16 --iters 200 --graph 20 --contiguous
$B --batch 16 --ctx 65536 --heads 128 --iters 20
