# One bench line per workload (device value, e2e, roofline), summarised.
T=${1:-bench}; O=gpurun_out/$T; mkdir -p $O
for w in gcd mul div div_fast ntt ntt_batch batch; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 ${BENCH_EXTRA} > $O/bench_$w.log 2>&1
  tail -1 $O/bench_$w.log | python -c '
import json,sys
try:
  d=json.loads(sys.stdin.read()); r=d["roofline"]
  print(d["config"]["workload"][:40].ljust(40), "%.4f ms" % d["ms_per_step"], "e2e %.4f ms" % d["e2e"]["ms_per_step"], "frac %.3f" % r["frac"], r.get("chain",{}).get("frac",""), d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
except Exception as e: print("ERR", e)' | tee -a $O/summary.txt
done
