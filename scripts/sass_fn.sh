#!/bin/bash
# Dump the SASS of one kernel (name regex) from an object: scripts/sass_fn.sh obj regex > out
obj=$1; re=$2
fn=$(cuobjdump -sass "$obj" | grep Function | sed 's/.*Function : //' | grep -E "$re" | head -1)
cuobjdump -sass -fun "$fn" "$obj" | grep -E '^\s+/\*[0-9a-f]{4}\*/' | sed 's@/\* 0x[0-9a-f]* \*/@@' | sed 's/ \+;.*$//' | sed 's/^ *//'
