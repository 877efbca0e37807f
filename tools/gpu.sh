#!/bin/bash
# run a command on the GPU box from the repo root (gpurun snapshots the cwd)
cd /root/repo || exit 1
T=${GPU_TIMEOUT:-1200}
timeout $((T + 1200)) /usr/local/graft/bin/gpurun --timeout "$T" -- "$@" 2>&1 | tail -2
