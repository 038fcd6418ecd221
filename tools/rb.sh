#!/bin/bash
# rebuild libflowreg_b200.so in-tree (incremental) from any cwd; build.py is
# loaded by path so a stale library cannot break the import
cd /root/repo && python -c "
import importlib.util, sys
spec = importlib.util.spec_from_file_location('_b', 'paper_2401_17493_b200/build.py')
m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m)
print(m.build(force='--force' in sys.argv))
" "$@" 2>&1 | tail -3
