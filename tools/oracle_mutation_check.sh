#!/usr/bin/env bash
# Mutation check of the oracle pins: each sed below injects a plausible mistake into a COPY of an
# oracle source and the CPU pin suite of that oracle must fail for every one.
#   atom_oracle.c (INT path): swapped nibbles, scatter instead of gather, truncation instead of
#     round-half-even, transposed scale index, dropped outlier group, wrong sign extension, wrong
#     level count, signed instead of absolute max
#   mx_oracle.c (Atom (FP), NEXT-2): swapped nibble packing, wrong E2M1 emax, floor(log2) off by
#     one, ties rounded down, no gather, sign dropped, E4M3 emax wrong
#   kv_oracle.c (KV cache, NEXT-3): 16 levels instead of 15, no zero point, floor instead of
#     rint, 1/d instead of 1/sqrt(d), swapped nibbles, block table ignored
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=$(mktemp -d)
cp -r "$ROOT/oracle" "$ROOT/synth" "$ROOT/tests" "$ROOT/pytest.ini" "$W"/
cd "$W"
M=(
'atom_oracle.c|test_oracle_pins.py|s/dst\[b\] = (uint8_t)((q\[2 \* b\] \& 0xF) | ((q\[2 \* b + 1\] \& 0xF) << 4));/dst[b] = (uint8_t)((q[2 * b + 1] \& 0xF) | ((q[2 * b] \& 0xF) << 4));/'
'atom_oracle.c|test_oracle_pins.py|s/xr\[jj\] = x\[r \* ldx + perm\[t \* ORACLE_GROUP + jj\]\];/xr[jj] = x[r * ldx + t * ORACLE_GROUP + jj];/'
'atom_oracle.c|test_oracle_pins.py|s/float r = nearbyintf(v);/float r = truncf(v);/'
'atom_oracle.c|test_oracle_pins.py|s/(double)a_scales\[t \* M + m\] \* (double)w_scales\[t \* N + n\]/(double)a_scales[m * G + t] * (double)w_scales[t * N + n]/'
'atom_oracle.c|test_oracle_pins.py|s/for (int64_t t = 0; t < G; ++t) {$/for (int64_t t = 0; t < G - (k_o ? 1 : 0); ++t) {/'
'atom_oracle.c|test_oracle_pins.py|s/return v >= 8 ? v - 16 : v;/return v >= 8 ? v - 15 : v;/'
'atom_oracle.c|test_oracle_pins.py|s/float levels = (float)((1 << nbits) - 1);/float levels = (float)((1 << (nbits - 1)) - 1);/'
'atom_oracle.c|test_oracle_pins.py|s/if (a > amax) amax = a;/if (xr[jj] > amax) amax = xr[jj];/'
'mx_oracle.c|test_oracle_pins_mx.py|s/else \*byte = (uint8_t)(\*byte | (c << 4));/else *byte = (uint8_t)((*byte << 4) | c);/'
'mx_oracle.c|test_oracle_pins_mx.py|s/oracle_mx_scale_byte(amax, is_fp4 ? 2 : 8)/oracle_mx_scale_byte(amax, is_fp4 ? 3 : 8)/'
'mx_oracle.c|test_oracle_pins_mx.py|s/int se = (E - 1) - emax_elem;/int se = E - emax_elem;/'
'mx_oracle.c|test_oracle_pins_mx.py|s/return (lo \& 1) ? lo + 1 : lo;/return lo;/'
'mx_oracle.c|test_oracle_pins_mx.py|s/const float a = fabsf(xr\[perm\[j\]\]);/const float a = fabsf(xr[j]);/'
'mx_oracle.c|test_oracle_pins_mx.py|s/return c | (signbit(x) ? 8 : 0);/return c;/'
'mx_oracle.c|test_oracle_pins_mx.py|s/oracle_mx_scale_byte(amax, is_fp4 ? 2 : 8)/oracle_mx_scale_byte(amax, is_fp4 ? 2 : 7)/'
'kv_oracle.c|test_oracle_pins_kv.py|s/const float s = range \/ 15.0f;/const float s = range \/ 16.0f;/'
'kv_oracle.c|test_oracle_pins_kv.py|s/const float u = (v\[i\] - mn) \* inv;/const float u = v[i] * inv;/'
'kv_oracle.c|test_oracle_pins_kv.py|s/float r = rintf(u);/float r = floorf(u);/'
'kv_oracle.c|test_oracle_pins_kv.py|s/const double scale = 1.0 \/ sqrt((double)d);/const double scale = 1.0 \/ (double)d;/'
'kv_oracle.c|test_oracle_pins_kv.py|s/const int q = (i \& 1) ? (c\[i \/ 2\] >> 4) : (c\[i \/ 2\] \& 15);/const int q = (i \& 1) ? (c[i \/ 2] \& 15) : (c[i \/ 2] >> 4);/'
'kv_oracle.c|test_oracle_pins_kv.py|s/const int64_t page = block_table\[b \* max_pages + t \/ KV_PAGE\], off = t % KV_PAGE;/const int64_t page = b * max_pages + t \/ KV_PAGE, off = t % KV_PAGE;/'
)
rc=0
for spec in "${M[@]}"; do
  f=${spec%%|*}; rest=${spec#*|}; t=${rest%%|*}; m=${rest#*|}
  cp "$ROOT/oracle/$f" "oracle/$f"
  sed -i "$m" "oracle/$f"
  if cmp -s "oracle/$f" "$ROOT/oracle/$f"; then echo "NOT APPLIED: $f $m"; rc=1; continue; fi
  rm -f oracle/liboracle.so
  if python -m pytest "tests/$t" -q >/dev/null 2>&1; then
    echo "SURVIVED: $f $m"; rc=1
  else
    echo "killed:   $f $m"
  fi
  cp "$ROOT/oracle/$f" "oracle/$f"
done
rm -rf "$W"
exit $rc
