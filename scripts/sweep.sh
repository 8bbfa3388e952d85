#!/bin/bash
# A/B sweep of SpMV kernel variants on the GPU box (one summary line per run).
#   CONFIGS="C2:1 C3:1"  VARIANTS="U4P0B4 U2P1B6"  POLS="x0s1 x1s1"
export PYTHONWARNINGS=ignore
out=${OUT:-gpurun_out/sweep.txt}
: > $out
for cfg in ${CONFIGS:-C2:1 C2:32 C3:1 C4:1}; do
  c=${cfg%%:*}; d=${cfg##*:}
  for lay in ${LAYOUTS:-compact}; do
  for v in ${VARIANTS:-U4P0B4 U2P1B6}; do
    for pol in ${POLS:-d}; do
      # pol "d" = the library defaults; "x<0|1>s<0|1>" forces the x / stream L2 policies
      if [ "$pol" = d ]; then unset ARGCSR_XPOL ARGCSR_SPOL; else export ARGCSR_XPOL=${pol:1:1} ARGCSR_SPOL=${pol:3:1}; fi
      # variant "K=V,K2=V2" = the default kernel with those environment settings
      for v_ in $(env | grep -o '^ARGCSR_[A-Z_0-9]*' | grep -v -e ARGCSR_XPOL -e ARGCSR_SPOL); do unset $v_; done
      vv=$v
      case $v in *=*) for kv in ${v//,/ }; do export "$kv"; done; vv=${ARGCSR_SPMV_VARIANT:-default};; esac
      r=$(ARGCSR_SPMV_VARIANT=$vv timeout 300 python bench.py --config $c --dcs $d --layout $lay --steps ${STEPS:-50} --warmup 5 --no-variants --no-cpu-baseline 2>/dev/null)
      python - "$c" "$d" "$v" "$pol" "$r" "$lay" >> $out <<'PY'
import json,sys
c,d,v,pol,r,lay=sys.argv[1:7]
try:
    j=json.loads(r); print(f"{c} dcs={d} {lay[:3]} {v.replace('ARGCSR_',''):7s} {pol} ms={j['ms_per_step']:.4f} GFLOP/s={j['value']:.1f} effGB/s={j['eff_GBps']:.0f} frac={j['roofline']['frac']:.3f} sm={j['clocks']['sm_mhz']}")
except Exception as e: print(c,d,v,pol,"FAILED",r[:200])
PY
    done
  done
  done
done
cat $out
