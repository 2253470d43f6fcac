#!/bin/bash
# Profiling recipe used for profiles/ (run under gpurun on one B200; see B200_PROFILING.md).
# 1) the plain run must exit 0; 2) launch list of one full timed C4 step (199 launches: guide
# derivative, bottom-link fill, support row + column, A1 fill, the row-strip plan's edge
# lengths and profiles (2 strips x 3 passes), prologue, 20 x [3 row, 3 column over the strips,
# 3 seam fix-ups] with iterations 2-20 taking the previous Eq. (3) step in their first row
# pass, and one closing update); 3) one `--set full` capture per kernel family (steady-state
# launches; k_row_pass launch 5 of a step is the first ROWUPD instance); 4) launch list of one
# eager C1 solve (302 launches) for the launch-gap breakdown (kernel time vs the event-timed
# solve).
# PART=c4 runs 1)-3), PART=extra runs 4)-5) (each part's outputs stay under gpurun's 64 MiB
# copy-back limit); unset runs both.
set -u
OUT=${OUT:-gpurun_out}
PART=${PART:-all}
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-extras"
if [ "$PART" != extra ]; then
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 199 -c 199 --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launches.log 2>&1
for spec in "k_col_cluster 4" "k_row_pass 2" "k_row_pass 4 row_update" "k_update 1" "k_guide_deriv 1" "k_prologue 1" "k_seam_fix 2"; do
  set -- $spec
  tag=${3:-$1}
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
      -o $OUT/full_$tag $CMD > $OUT/ncu_full_$tag.log 2>&1
done
fi
if [ "$PART" != c4 ]; then
# 5) C3 (8 x 4K, C_t = 3) in one batched context, one iteration per solve (tools/c3_batch.py):
#    the launch list of create + five solves, and one --set full capture each of a column pass
#    (launch 10 of k_col_cluster: after the 8 per-image support passes and the first) and a row
#    pass (launch 3 of k_row_pass: after the support pass and the first)
C3_ITERS=1 python tools/c3_batch.py > $OUT/c3_once.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv \
    --log-file $OUT/c3_launches.csv env C3_ITERS=1 python tools/c3_batch.py > $OUT/ncu_c3.log 2>&1
for spec in "k_col_cluster 9" "k_row_pass 2"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 -s $2 -c 1 \
      -o $OUT/full_c3_$1 env C3_ITERS=1 python tools/c3_batch.py > $OUT/ncu_full_c3_$1.log 2>&1
done
python tools/c1_once.py > $OUT/c1_once.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 307 -c 302 --csv --log-file $OUT/c1_launches.csv \
    python tools/c1_once.py > $OUT/ncu_c1.log 2>&1
fi
echo done
