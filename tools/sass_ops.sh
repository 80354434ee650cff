#!/bin/bash
# static SASS opcode histogram of one kernel: tools/sass_ops.sh <object> <mangled-name-substring>
cuobjdump -sass "$1" | awk -v k="$2" '/Function :/{f=index($0,k)>0} f' | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed -E 's/^\s+\/\*[0-9a-f]+\*\/\s+(@!?U?P[0-9T] )?//' | awk '{print $1}' | sed 's/\..*//;s/;//' | sort | uniq -c | sort -rn | head -${3:-30}
