for v in A B C D; do echo "== variant $v"; DOGIP_LIB=paper_1710_09913_b200/libdogip_$v.so python scripts/config_sweep.py --configs C2p4,C3,C4,C5 --iso --iters 10 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(f\"{r['config']:5s} {r['form']:7s} apply {r['apply_ms']:8.3f} ms  frac {r['frac_measured']:.3f}  fp64 {r['fp64_TFs']:.1f} TF/s  cg {r['cg_ms_per_iter']:.3f}\")
"; done
