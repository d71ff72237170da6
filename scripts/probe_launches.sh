OUT=gpurun_out/$1; mkdir -p $OUT
for wk in "C3 symmetric" "C4 ranking"; do
  set -- $wk
  python scripts/fit_probe.py $1 $2 20 3 >> $OUT/probe.jsonl 2>>$OUT/err.log
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launch_$1_$2.csv python scripts/fit_probe.py $1 $2 4 1 > /dev/null 2>>$OUT/err.log
done
cat $OUT/probe.jsonl
