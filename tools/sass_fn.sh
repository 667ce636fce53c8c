#!/bin/bash
# SASS of one kernel of a built library: sass_fn.sh LIB.so NAME_REGEX > out.sass
cuobjdump -sass "$1" | awk -v re="$2" '/Function : /{p = ($0 ~ re)} p'
