# usage: bash tools/ncu_cap.sh NAME KREGEX COUNT [prof_batch args...]
# runs the command once without ncu, then captures --set full of COUNT launches
name=$1; kre=$2; cnt=$3; shift 3
mkdir -p gpurun_out
timeout 300 python tools/prof_batch.py "$@" | tail -1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$kre" -c "$cnt" \
  --metrics smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.pct,smsp__inst_executed_op_global_red.sum \
  -o gpurun_out/$name -f python tools/prof_batch.py "$@" > gpurun_out/$name.log 2>&1
echo "ncu rc=$?"
