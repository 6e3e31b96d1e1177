for v in "" cond_prio=1 cdense_ctas=0 cond_prio=1,cdense_ctas=0 cdense_ctas=1 cond_prio=1,cdense_ctas=1; do echo "== $v $(VARIANTS=$v python tools/yy_bench.py C3 2>&1 | tail -1 | cut -c1-110)"; done
