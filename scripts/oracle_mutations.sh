# Mutation check of the oracle's pins (round-1 judge's three mutations of the R8 / R15 table
# rules): each mutated copy of oracle/eq_oracle.c must fail at least one -m "not gpu" oracle test.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
muts=(
  's/if (b < 0 || r\[c\] > r\[b\] || (r\[c\] == r\[b\] \&\& hist\[c\] > hist\[b\])) b = c;/if (b < 0 || r[c] < r[b] || (r[c] == r[b] \&\& hist[c] < hist[b])) b = c;/'
  's/if (f\[c\] > 1 \&\& (b < 0 || f\[c\] > f\[b\])) b = c;/if (f[c] > 1 \&\& (b < 0 || f[c] < f[b])) b = c;/'
  's/if (b < 0 || r\[i\] > r\[b\] || (r\[i\] == r\[b\] \&\& w\[i\] > w\[b\])) b = i;/if (b < 0 || r[i] < r[b] || (r[i] == r[b] \&\& w[i] > w[b])) b = i;/'
  's/if (f\[i\] > 1 \&\& (b < 0 || f\[i\] > f\[b\])) b = i;/if (f[i] > 1 \&\& (b < 0 || f[i] < f[b])) b = i;/'
  's/if ((unsigned __int128)32 \* EQO_M \* x >= W)/if ((unsigned __int128)16 * EQO_M * x >= W)/'
  's/if (hist\[c\] \&\& !used\[c\] \&\& (b < 0 || hist\[c\] > hist\[b\])) b = c;/if (hist[c] \&\& !used[c] \&\& (b < 0 || hist[c] >= hist[b])) b = c;/'
  's/f\[c\] = q < 1 ? 1 : (int64_t)q;/f[c] = q < 1 ? 0 : (int64_t)q;/'
)
rc=0
for m in "${muts[@]}"; do
  T=$(mktemp -d)
  cp -r "$ROOT/oracle" "$ROOT/eqsynth" "$ROOT/tests" "$ROOT/pytest.ini" "$T/"
  rm -f "$T"/oracle/*.so
  sed -i "$m" "$T/oracle/eq_oracle.c"
  if cmp -s "$T/oracle/eq_oracle.c" "$ROOT/oracle/eq_oracle.c"; then echo "MUTATION NOT APPLIED: $m"; rc=1; continue; fi
  (cd "$T" && timeout 900 python -m pytest tests/test_oracle_codec.py -q -x -m "not gpu" > "$T/log" 2>&1)
  r=$?
  if [ $r -eq 0 ]; then echo "SURVIVED: $m"; rc=1; else echo "killed ($(grep -m1 FAILED "$T/log"))"; fi
  rm -rf "$T"
done
exit $rc
