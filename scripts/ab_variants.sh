#!/bin/bash
# A/B of experimental builds: bash scripts/ab_variants.sh "base S6 G2" [configs]
VARIANTS=${1:-base}
CONFIGS=${2:-C2p4,C3,C4,C5}
for v in $VARIANTS; do
  echo "== variant $v"
  if [ "$v" = "base" ]; then LIBP=paper_1710_09913_b200/libdogip.so; else LIBP=paper_1710_09913_b200/libdogip_$v.so; fi
  DOGIP_LIB=$LIBP python scripts/config_sweep.py --configs $CONFIGS --iso --iters 10 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(f\"{r['config']:5s} {r['form']:7s} apply {r['apply_ms']:8.3f} ms  frac {r['frac_measured']:.3f}  fp64 {r['fp64_TFs']:.1f} TF/s  cg {r['cg_ms_per_iter']:.3f}\")
"
done
