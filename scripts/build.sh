#!/bin/bash
# build the sm_100a library; print the tail of the log and fail loudly on error
cd "$(dirname "$0")/.." && python -m paper_2506_17626_b200.build --force > /tmp/fl_build.log 2>&1 || { grep -E "error|Error" /tmp/fl_build.log | head -20; exit 1; }
tail -1 /tmp/fl_build.log
