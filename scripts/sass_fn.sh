#!/bin/bash
# Dump the SASS of the first function in an object whose name matches a regex (one instruction per line)
#   scripts/sass_fn.sh <obj> <regex>
fn=$(cuobjdump -sass "$1" | grep -E "Function : " | awk '{print $3}' | grep -E "$2" | head -1)
cuobjdump -sass -fun "$fn" "$1" | grep -E "^\s+/\*[0-9a-f]+\*/" | sed 's@/\*[0-9a-f]*\*/@@; s@;.*@@'
