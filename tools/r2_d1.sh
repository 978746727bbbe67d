# INT4 encode: packed statistics / folded NaN check / LEA nibble packing; parity + per-item timing
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for r in 1 2; do for s in INT4 INT8 GSE8; do echo "$s $(timeout 120 python tools/prof_quant.py $s 64 2>&1 | tail -1)"; done; done
