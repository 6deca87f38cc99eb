#!/bin/bash
# SASS of the kernels matching a regex in an object / library: tools/sass_of.sh <file> <regex> > out.sass
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : / {f = ($0 ~ pat)} f' \
  | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed -E 's@^\s+/\*([0-9a-f]+)\*/\s+@\1 @; s@\s*/\*.*@@; s@ ;$@@'
