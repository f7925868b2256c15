#!/bin/bash
# Host-side diagnosis of a GPU box: memory, THP, NUMA, storage, and the D2H/H2D
# rate across a large registered image.  Output: gpurun_out/diag/.
OUT=gpurun_out/diag; mkdir -p $OUT
{ nproc; free -g; lscpu | head -25; cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag;
  numactl --hardware 2>&1 | head; df -h / /tmp /dev/shm $GRAFT_REPO_ROOT 2>&1; mount | grep -E " / | /tmp | /dev/shm " ; lsblk 2>&1 | head -20;
  nvidia-smi -q | grep -iE "link|gen|width" | head -20; } > $OUT/sys.txt 2>&1
timeout 600 ./tools/probe/probe_bigpin ${BIGPIN_GIB:-120} 16 > $OUT/bigpin.txt 2>&1
for d in /tmp $GRAFT_REPO_ROOT /dev/shm; do timeout 300 ./tools/probe/probe_io $d ${IO_GIB:-16} 8 16 >> $OUT/io.txt 2>&1; done
