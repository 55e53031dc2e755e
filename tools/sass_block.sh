#!/bin/bash
# print the SASS of a kernel of libising.so: tools/sass_block.sh <cubin-name> [pattern-start] [n]
so=${SO:-/root/repo/paper_2311_09275_b200/lib/libising.so}
cd /tmp && cuobjdump -xelf $1.sm_100a.cubin $so > /dev/null && nvdisasm -c $1.sm_100a.cubin | grep -E "^\s+/\*[0-9a-f]+\*/|^\.L" | sed 's/^ *//' > /tmp/$1.sass
wc -l < /tmp/$1.sass
