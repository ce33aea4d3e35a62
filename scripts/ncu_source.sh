#!/bin/bash
# Per-instruction stall samples of one kernel (SASS page), small enough to copy back:
#   bash scripts/ncu_source.sh REGEX OUT_PREFIX -- command...
RX=$1; OUT=$2; shift 3
"$@" > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$RX" -s 1 -c 1 -o "$OUT" "$@" > "$OUT.log" 2>&1
ncu -i "$OUT.ncu-rep" --page source --csv --print-source sass > "$OUT.sass.csv" 2>/dev/null
ncu -i "$OUT.ncu-rep" --page raw --csv > "$OUT.raw.csv" 2>/dev/null
rm -f "$OUT.ncu-rep"
