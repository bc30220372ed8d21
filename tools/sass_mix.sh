#!/bin/bash
# usage: tools/sass_mix.sh file.cubin pattern  -- opcode histogram of the first kernel whose name matches
fn=$(cuobjdump -sass "$1" | grep "Function" | grep "$2" | head -1 | sed 's/.*Function : //')
echo "$fn"
cuobjdump -sass -fun "$fn" "$1" | grep -E "^\s+/\*[0-9a-f]+\*/" | sed -E 's/^\s+\/\*[0-9a-f]+\*\/\s+//' | sed -E 's/^@!?U?P[0-9T]+\s+//' | awk '{print $1}' | sed 's/\..*//' | sort | uniq -c | sort -rn | head -${3:-12}
