#!/bin/bash
# SASS of one kernel of a built .so: tools/sass_fn.sh LIB PATTERN (e.g. 'macko_spmvILi10ELi4ELi1E')
lib=$1; pat=$2
cuobjdump -sass "$lib" | awk -v p="$pat" '/Function :/ {on = index($0, p) > 0} on' | sed 's@/\* 0x[0-9a-f]* \*/@@' | grep -E '^\s+/\*[0-9a-f]{4,}\*/' 
