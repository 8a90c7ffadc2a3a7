#!/usr/bin/env bash
# Mutation check of the oracle pins: each sed below injects a plausible mistake into a COPY of
# oracle/atom_oracle.c (swapped nibbles, scatter instead of gather, truncation instead of
# round-half-even, transposed scale index, dropped outlier group, wrong sign extension, wrong
# level count, signed instead of absolute max) and the CPU pin suite must fail for every one.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
W=$(mktemp -d)
cp -r "$ROOT/oracle" "$ROOT/synth" "$ROOT/tests" "$ROOT/pytest.ini" "$W"/
cd "$W"
M=(
's/dst\[b\] = (uint8_t)((q\[2 \* b\] \& 0xF) | ((q\[2 \* b + 1\] \& 0xF) << 4));/dst[b] = (uint8_t)((q[2 * b + 1] \& 0xF) | ((q[2 * b] \& 0xF) << 4));/'
's/xr\[jj\] = x\[r \* ldx + perm\[t \* ORACLE_GROUP + jj\]\];/xr[jj] = x[r * ldx + t * ORACLE_GROUP + jj];/'
's/float r = nearbyintf(v);/float r = truncf(v);/'
's/(double)a_scales\[t \* M + m\] \* (double)w_scales\[t \* N + n\]/(double)a_scales[m * G + t] * (double)w_scales[t * N + n]/'
's/for (int64_t t = 0; t < G; ++t) {$/for (int64_t t = 0; t < G - (k_o ? 1 : 0); ++t) {/'
's/return v >= 8 ? v - 16 : v;/return v >= 8 ? v - 15 : v;/'
's/float levels = (float)((1 << nbits) - 1);/float levels = (float)((1 << (nbits - 1)) - 1);/'
's/if (a > amax) amax = a;/if (xr[jj] > amax) amax = xr[jj];/'
)
rc=0
for m in "${M[@]}"; do
  cp "$ROOT/oracle/atom_oracle.c" oracle/atom_oracle.c
  sed -i "$m" oracle/atom_oracle.c
  if cmp -s oracle/atom_oracle.c "$ROOT/oracle/atom_oracle.c"; then echo "NOT APPLIED: $m"; rc=1; continue; fi
  rm -f oracle/liboracle.so
  if python -m pytest tests/test_oracle_pins.py -q >/dev/null 2>&1; then
    echo "SURVIVED: $m"; rc=1
  else
    echo "killed:   $m"
  fi
done
rm -rf "$W"
exit $rc
