for v in 16 32 64 112 1; do timeout -s KILL 30 ./tools/microbench/mb11 $v 2>&1 | tail -7; done
