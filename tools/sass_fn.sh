#!/bin/bash
# usage: tools/sass_fn.sh <mangled-substring>  -> SASS of the matching function(s) of liblbpfused.so
cuobjdump -sass /root/repo/paper_1504_01883_b200/liblbpfused.so | awk -v pat="$1" '/Function : /{f=($0 ~ pat)} f'
