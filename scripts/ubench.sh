#!/bin/bash
cd "$(dirname "$0")"
for m in 0 1; do for w in 4 8; do for s in 2 4 6; do
  timeout -s KILL 30 ./ubench_gather $m $s 1 131072 1 $w 1
done; done; done
timeout -s KILL 30 ./ubench_gather 0 4 1 8192 1 4 1
timeout -s KILL 30 ./ubench_gather 1 4 1 8192 1 4 1
timeout -s KILL 30 ./ubench_gather 0 3 2 131072 1 4 1
timeout -s KILL 30 ./ubench_gather 1 3 2 131072 1 4 1
