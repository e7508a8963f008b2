#!/bin/bash
# registers / spills of the kernels in an object whose demangled name matches $2: regs.sh build/x.o 'regex'
cuobjdump -res-usage "$1" 2>/dev/null | awk '/Function/{f=$0; next} /REG:/{print $0 "\t" f}' | c++filt | \
  sed -E 's/.*REG:([0-9]+) STACK:([0-9]+).*Function (.*):$/\1 \2 \3/; s/rgnn::\(anonymous namespace\):://' | grep -E "$2" | cut -c1-160
