#!/bin/bash
# retry a gpurun call until it is not transient: $1 = log name, rest = command
name=$1; shift
for i in $(seq 1 20); do
  timeout 3600 /usr/local/graft/bin/gpurun --timeout 2400 -- "$@" > gpurun_out/${name}_call.log 2>&1
  if ! grep -q "status=transient" gpurun_out/${name}_call.log; then break; fi
  sleep 150
done
