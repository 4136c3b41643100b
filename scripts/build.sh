#!/bin/bash
# build everything; non-zero exit on any compile error (use before gpurun)
set -e
cd "$(dirname "$0")/.."
python -c "
import sys; sys.path.insert(0,'.')
import __graft_entry__ as g; g.build()"
