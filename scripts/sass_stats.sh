#!/bin/bash
# Per-kernel SASS instruction counts (total, R2UR, ELECT, UTCHMMA) for a built object:
#   scripts/sass_stats.sh paper_2605_11111_b200/csrc/build/conv_tc.o [regex]
obj=$1; pat=${2:-.}
cuobjdump -sass "$obj" | awk -v pat="$pat" '
/Function :/ { if (name != "" && name ~ pat) printf "%-90s total=%5d R2UR=%4d ELECT=%3d UTCHMMA=%4d\n", name, tot, r2u, el, mm;
               name=$3; tot=0; r2u=0; el=0; mm=0; next }
/^ +\/\*[0-9a-f]+\*\// { tot++; if ($0 ~ /R2UR/) r2u++; if ($0 ~ /ELECT/) el++; if ($0 ~ /UTC[A-Z]*MMA/) mm++ }
END { if (name != "" && name ~ pat) printf "%-90s total=%5d R2UR=%4d ELECT=%3d UTCHMMA=%4d\n", name, tot, r2u, el, mm }' | sed 's/_ZN2dp43_GLOBAL__N__[0-9a-f_]*//'
