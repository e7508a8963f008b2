#!/bin/bash
# A clean copy of a commit (default HEAD) in ab_head/ for `gpu_run.sh abhead` (git-ignored; travels with gpurun)
set -e
rm -rf ab_head && mkdir ab_head
git archive "${1:-HEAD}" | tar -x -C ab_head
