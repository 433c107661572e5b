#!/bin/bash
cd "$(dirname "$0")"
# build the microbenchmarks (binaries are not tracked)
for b in ubench_gather ubench_mma ubench_mma2 ubench_mcast ubench_alu ubench_tmem; do
  [ -x $b ] || nvcc -std=c++17 -O3 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -o $b $b.cu -lcuda
done
for m in 0 1; do for w in 4 8; do for s in 2 4 6; do
  timeout -s KILL 30 ./ubench_gather $m $s 1 131072 1 $w 1
done; done; done
timeout -s KILL 30 ./ubench_gather 0 4 1 8192 1 4 1
timeout -s KILL 30 ./ubench_gather 1 4 1 8192 1 4 1
timeout -s KILL 30 ./ubench_gather 0 3 2 131072 1 4 1
timeout -s KILL 30 ./ubench_gather 1 3 2 131072 1 4 1
