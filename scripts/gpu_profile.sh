#!/bin/bash
# per-kernel DRAM traffic of one step of each config in CFGS (ncu metrics, clock-control none)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for CFG in ${CFGS:-C2}; do
  timeout 600 python scripts/profile_step.py --config $CFG --bulk > gpurun_out/step_$CFG.log 2>&1 || { tail gpurun_out/step_$CFG.log; continue; }
  K='regex:k_hist|k_onesweep|k_segscan|k_ev_pos|k_epoch_stats|k_sweep|k_score|k_key_belady|k_select|k_fill_stream|k_place'
  [ "$CFG" != "C5" ] && K="$K|k_replay"
  timeout 2400 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
     --clock-control none --csv -k "$K" --log-file gpurun_out/traffic_$CFG.csv \
     python scripts/profile_step.py --config $CFG --bulk > gpurun_out/ncu_step_$CFG.log 2>&1
  python scripts/ncu_traffic.py gpurun_out/traffic_$CFG.csv $CFG
done
cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json
