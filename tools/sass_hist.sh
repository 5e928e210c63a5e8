#!/bin/bash
# usage: tools/sass_hist.sh <mangled-kernel-name> [lib]  -> static SASS opcode histogram
lib=${2:-paper_1510_03560_b200/libplbm_gpu.so}
cuobjdump -sass "$lib" | awk -v f="Function : $1" '$0 ~ f {p=1;next} /Function :/{p=0} p' > /tmp/k.sass
grep -oP '^\s+/\*[0-9a-f]+\*/\s+(@!?U?P[T0-9]\s+)?\K[A-Z0-9_]+' /tmp/k.sass | sort | uniq -c | sort -rn | head -${3:-25}
