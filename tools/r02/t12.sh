timeout -s KILL 30 ./tools/microbench/mb12 0; timeout -s KILL 30 ./tools/microbench/mb12 1
