#!/bin/bash
# rebuild libflowreg_b200.so in-tree (incremental) from any cwd
cd /root/repo && python -m paper_2401_17493_b200.build "$@" 2>&1 | tail -3
