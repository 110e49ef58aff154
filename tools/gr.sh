#!/bin/bash
# gpurun from the repository root (the snapshot is taken from the cwd)
cd "$(dirname "$0")/.." && exec /usr/local/graft/bin/gpurun "$@"
