M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg.per_second,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,sm__inst_executed_pipe_uniform.sum,smsp__warps_issue_stalled_barrier_per_warp_active.pct,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum
for v in nsb2 seq2; do
  ncu --metrics $M --clock-control none -k regex:flashsign -s 1 -c 1 --csv python tests/run_variant.py $v c5 2 2>/dev/null | grep -v "^==" | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin):
  if len(r)>12 and r[0]!='ID': print('$v', r[-3], r[-1])
"
done
