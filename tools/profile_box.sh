#!/bin/bash
# One GPU call: tools/profile_round.sh, then the ncu summaries written on the
# box (profiles/<tag>_*.md, profiles/ncu_summary.json copied to gpurun_out/
# for the merge back) and the large .ncu-rep files dropped (64 MiB merge cap).
# usage: tools/profile_box.sh <tag> <scene>
TAG=${1:-r02e}; SC=${2:-c5}
bash tools/profile_round.sh $SC > gpurun_out/profile_round.log 2>&1
REPS=$(ls gpurun_out/prof_*_$SC.ncu-rep | tr '\n' ',' | sed 's/,$//')
python tools/ncu_summary.py $TAG $SC gpurun_out/launches_$SC.csv $REPS gpurun_out/prof_driver_pcg_$SC.log \
  gpurun_out/evalflops_$SC.csv > gpurun_out/ncu_summary.log 2>&1
mkdir -p gpurun_out/profiles
cp profiles/${TAG}_*_$SC.md profiles/ncu_summary.json gpurun_out/profiles/
for f in gpurun_out/prof_*_$SC.ncu-rep; do
  [ $(stat -c %s $f) -gt 12000000 ] && rm -f $f
done
du -sh gpurun_out
tail -3 gpurun_out/ncu_summary.log
