# per-variant ncu (one k_sweep launch, 512 C5 scenes): executed instructions, IPC, stall split
mkdir -p gpurun_out/r02
for lib in scratch/libs/*.so; do
  n=$(basename $lib .so)
  CA_LIBRARY=$PWD/$lib ncu --section WarpStateStats --section ComputeWorkloadAnalysis --section LaunchStats --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__pcsamp_warps_issue_stalled_no_instructions.sum,smsp__pcsamp_sample_count.sum --clock-control none -k regex:k_sweep --launch-skip 2 --launch-count 1 --csv --page raw python profiles/prof_driver.py 512 3 > gpurun_out/r02/ncu_ab_$n.csv 2> gpurun_out/r02/ncu_ab_$n.err
  echo "$n rc=$?"
done
