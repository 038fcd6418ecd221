#!/bin/bash
# Event-time the default library and every build variant under
# paper_2401_17493_b200/_variants/ (gather, matvec, refresh at 256^3).
cd "$(dirname "$0")/.."
python tools/gather_time.py 2>&1 | tail -1
for v in paper_2401_17493_b200/_variants/*.so; do
  FRG_LIB=$v python tools/gather_time.py 2>&1 | tail -1
done
