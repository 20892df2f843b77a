#!/bin/bash
# Runs a command in the background; if its log stops growing for ~20 s,
# attaches cuda-gdb to dump the running kernels / blocks, then kills it.
#   tools/hang_catch.sh <tag> <cmd...>
tag=$1; shift
log=gpurun_out/hc_$tag.log
"$@" > $log 2>&1 &
pid=$!
last=-1; still=0
while kill -0 $pid 2>/dev/null; do
  sleep 5
  sz=$(stat -c %s $log)
  if [ "$sz" = "$last" ]; then still=$((still+1)); else still=0; fi
  last=$sz
  if [ $still -ge 4 ]; then
    echo "stalled; attaching cuda-gdb" >> $log
    timeout 240 cuda-gdb -p $pid -batch -ex "info cuda kernels" -ex "info cuda blocks" \
      -ex "info cuda warps" -ex "bt" -ex "cuda kernel 1" -ex "info cuda blocks" \
      -ex "info cuda warps" -ex "info cuda lanes" -ex "bt" -ex "info cuda sms" \
      > gpurun_out/hc_${tag}_gdb.txt 2>&1
    py-spy dump --pid $pid > gpurun_out/hc_${tag}_py.txt 2>&1
    kill -9 $pid
    echo "HANG" >> $log
    break
  fi
done
wait $pid 2>/dev/null
echo "rc=$?" >> $log
