# Mutation check of the oracle's pins (the round-1 judge's mutations of the R8 / R15 table rules,
# plus round-2 mutations of the quantiser, Q†, row chunking, the escape order and R18's group
# order): each mutated
# copy of oracle/eq_oracle.c must fail at least one -m "not gpu" oracle test.
set -u
ROOT=$(cd "$(dirname "$0")/.." && pwd)
ONLY=${ONLY:-}            # e.g. ONLY=13 runs mutations 13.. only
muts=(
  's/if (b < 0 || r\[c\] > r\[b\] || (r\[c\] == r\[b\] \&\& hist\[c\] > hist\[b\])) b = c;/if (b < 0 || r[c] < r[b] || (r[c] == r[b] \&\& hist[c] < hist[b])) b = c;/'
  's/if (f\[c\] > 1 \&\& (b < 0 || f\[c\] > f\[b\])) b = c;/if (f[c] > 1 \&\& (b < 0 || f[c] < f[b])) b = c;/'
  's/if (b < 0 || r\[i\] > r\[b\] || (r\[i\] == r\[b\] \&\& w\[i\] > w\[b\])) b = i;/if (b < 0 || r[i] < r[b] || (r[i] == r[b] \&\& w[i] > w[b])) b = i;/'
  's/if (f\[i\] > 1 \&\& (b < 0 || f\[i\] > f\[b\])) b = i;/if (f[i] > 1 \&\& (b < 0 || f[i] < f[b])) b = i;/'
  's/if ((unsigned __int128)32 \* EQO_M \* x >= W)/if ((unsigned __int128)16 * EQO_M * x >= W)/'
  's/if (hist\[c\] \&\& !used\[c\] \&\& (b < 0 || hist\[c\] > hist\[b\])) b = c;/if (hist[c] \&\& !used[c] \&\& (b < 0 || hist[c] >= hist[b])) b = c;/'
  's/f\[c\] = q < 1 ? 1 : (int64_t)q;/f[c] = q < 1 ? 0 : (int64_t)q;/'
  # round 2: bf16 RNE tie rule, E4M3 tie rule, clamp bound, subnormal boundary (quantiser, Q†)
  's/else p = (lo \& 1) ? hi : lo; /else p = hi; /'
  's/q = ldexp(rint(m \* 16.0), k - 4);/q = ldexp(round(m * 16.0), k - 4);/'
  's/if (r > 448.0) r = 448.0;/if (r > 480.0) r = 480.0;/'
  's/if (a < ldexp(1.0, -6)) {/if (a < ldexp(1.0, -7)) {/'
  # row chunking (R16) collapsed to flat chunking
  's/return s \* seg + j \* cs;/return k * cs;/'
  # the escape's two singles in the opposite order, consistently in encoder and decoder (a
  # self-consistent wire-format change that round trips: only the hand-derived streams see it)
  '/eqo_w_put(\&x, freq\[b\], cum\[b\], tmp, \&pos);/{N;s/eqo_w_put(\&x, freq\[b\], cum\[b\], tmp, \&pos);\n\( *\)eqo_w_put(\&x, freq\[a\], cum\[a\], tmp, \&pos);/eqo_w_put(\&x, freq[a], cum[a], tmp, \&pos);\n\1eqo_w_put(\&x, freq[b], cum[b], tmp, \&pos);/};s/sym\[2 \* i + k\] = (uint8_t)s;/sym[2 * i + 1 - k] = (uint8_t)s;/'
  # R18 (session 3), each self-consistent in encoder and decoder: 32-symbol groups; escaped
  # positions patched in decreasing order; an escaped pair's codes in the order b, a
  's/#define EQO_GROUP 16/#define EQO_GROUP 32/'
  's|for (int64_t i = 0; i < g / 2; i++) {                         /\* (2) \*/|for (int64_t i = g / 2 - 1; i >= 0; i--) {                     /* (2) */|'
  's/sf\[m\] = freq\[a\]; sc\[m\] = cum\[a\]; m++;/sf[m] = freq[b]; sc[m] = cum[b]; m++; sf[m] = freq[a]; sc[m] = cum[a]; m++; continue;/;s/if (eqo_w_single(\&x, freq, cum, in, nbytes, \&p, \&sym\[g0 + 2 \* i\])) return 2;/if (eqo_w_single(\&x, freq, cum, in, nbytes, \&p, \&sym[g0 + 2 * i + 1])) return 2; if (eqo_w_single(\&x, freq, cum, in, nbytes, \&p, \&sym[g0 + 2 * i])) return 2; continue;/'
)
rc=0
i=0
for m in "${muts[@]}"; do
  i=$((i + 1)); if [ -n "$ONLY" ] && [ $i -lt $ONLY ]; then continue; fi
  T=$(mktemp -d)
  cp -r "$ROOT/oracle" "$ROOT/eqsynth" "$ROOT/tests" "$ROOT/pytest.ini" "$T/"
  rm -f "$T"/oracle/*.so
  sed -i "$m" "$T/oracle/eq_oracle.c"
  if cmp -s "$T/oracle/eq_oracle.c" "$ROOT/oracle/eq_oracle.c"; then echo "MUTATION NOT APPLIED: $m"; rc=1; continue; fi
  (cd "$T" && timeout 1200 python -m pytest tests/test_oracle_codec.py tests/test_oracle_quant.py -q -x -m "not gpu" > "$T/log" 2>&1)
  r=$?
  if [ $r -eq 0 ]; then echo "SURVIVED: $m"; rc=1; else echo "killed ($(grep -m1 FAILED "$T/log"))"; fi
  rm -rf "$T"
done
exit $rc
