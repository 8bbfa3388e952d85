for xr in on off; do
python - $xr <<'PY' > gpurun_out/c3_$1.txt 2>&1
import sys
PY
done
cat > /tmp/c3prof.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1203_5737_b200 as argcsr
from paper_1203_5737_b200 import synthetic
xr = sys.argv[1]
A = synthetic.rmat(24, 16, 1, torch.device('cuda'))
m = argcsr.argcsr_from_torch(A.num_rows, A.num_cols, A.row_pointers, A.columns, A.values, 128, 1, x_remap=xr)
x = synthetic.bench_input(A.num_cols, torch.device('cuda'), torch.float64)
y = torch.empty(A.num_rows, dtype=torch.float64, device='cuda')
for _ in range(5): argcsr.spmv_torch(m, x, out=y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): argcsr.spmv_torch(m, x, out=y)
e1.record(); torch.cuda.synchronize()
print(xr, 'x_remap', m.x_remap, 'used', m.x_used_columns, 'ms', e0.elapsed_time(e1)/20)
PY
for xr in on off; do python /tmp/c3prof.py $xr; done
for xr in on off; do ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum -k regex:spmv_ -s 10 -c 3 --csv python /tmp/c3prof.py $xr 2>/dev/null | grep -v "^==" | tail -12; done
