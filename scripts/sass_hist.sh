#!/bin/bash
# Opcode histogram of one band4 variant: sass_hist.sh <template-args-mangled> [lib]
LIB=${2:-paper_1612_00746_b200/lib/libctqw.so}
cuobjdump -sass -fun "_ZN4ctqw2b412band4_kernel${1}EEvNS0_9Band4ArgsE" $LIB 2>/dev/null | grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9_.]+" | awk '{print $2}' | sort | uniq -c | sort -rn
