#!/bin/bash
# Run one gpurun call after any in-flight call finished: tools/gpu.sh <timeout_s> '<command>'
T=$1; shift
while /usr/local/graft/bin/gpurun --status 2>/dev/null | grep -q '"in_flight": 1'; do sleep 10; done
exec /usr/local/graft/bin/gpurun --timeout "$T" -- "$@"
