#!/bin/bash
# A/B sweep of SpMV kernel variants on the GPU box (one summary line per run).
#   CONFIGS="C2:1 C3:1"  VARIANTS="U4P0B4 U2P1B6"  POLS="x0s1 x1s1"
export PYTHONWARNINGS=ignore
out=${OUT:-gpurun_out/sweep.txt}
: > $out
for cfg in ${CONFIGS:-C2:1 C2:32 C3:1 C4:1}; do
  c=${cfg%%:*}; d=${cfg##*:}
  for v in ${VARIANTS:-U4P0B4 U2P1B6}; do
    for pol in ${POLS:-x0s1}; do
      xp=${pol:1:1}; sp=${pol:3:1}
      r=$(ARGCSR_XPOL=$xp ARGCSR_SPOL=$sp ARGCSR_SPMV_VARIANT=$v timeout 300 python bench.py --config $c --dcs $d --steps ${STEPS:-50} --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null)
      python - "$c" "$d" "$v" "$pol" "$r" >> $out <<'PY'
import json,sys
c,d,v,pol,r=sys.argv[1:6]
try:
    j=json.loads(r); print(f"{c} dcs={d} {v:7s} {pol} ms={j['ms_per_step']:.4f} GFLOP/s={j['value']:.1f} effGB/s={j['eff_GBps']:.0f} frac={j['roofline']['frac']:.3f} sm={j['clocks']['sm_mhz']}")
except Exception as e: print(c,d,v,pol,"FAILED",r[:200])
PY
    done
  done
done
cat $out
