#!/bin/bash
set -x
nproc; free -g; lscpu | head -30; nvidia-smi; nvidia-smi topo -m; numactl --hardware 2>&1 | head -20
ulimit -l
timeout 600 ./tools/probe/probe_box 2>&1
