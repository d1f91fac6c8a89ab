# The round's profile set (one GPU box): launch list of three eager C2 trees,
# ncu --set full of the hot kernels (CSV pages), the combined timeline.
#   bash tools/profile_round.sh TAG      -> gpurun_out/TAG_*
tag=$1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_c2.csv \
  python tools/probe.py c2eager > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/${tag}_launches_c2.csv > gpurun_out/${tag}_launch_summary.txt
bash tools/ncu_capture.sh gpurun_out/${tag}_ncu_count_l6 k_count_fused 6 c2eager
bash tools/ncu_capture.sh gpurun_out/${tag}_ncu_count_l3 k_count_fused 3 c2eager
bash tools/ncu_capture.sh gpurun_out/${tag}_ncu_part_l6 k_partition_split 5 c2eager
bash tools/ncu_capture.sh gpurun_out/${tag}_ncu_oaa_early_l6 k_oaa_early 4 c2eager
bash tools/ncu_capture.sh gpurun_out/${tag}_ncu_hcpre_l5 k_hc_pre 5 c2eager
bash tools/ncu_capture.sh gpurun_out/${tag}_ncu_hcpost_l5 k_hc_post_finish 5 c2eager
bash tools/ncu_capture.sh gpurun_out/${tag}_ncu_prep8 k_prep8 0 c2eager
bash tools/ncu_capture.sh gpurun_out/${tag}_ncu_walk_c3 k_walk 3 walk
GT_COUNT_TS=1 GT_HC_TIMING=1 python tools/probe.py tl > gpurun_out/${tag}_timeline_c2.txt 2>&1
