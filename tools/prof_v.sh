#!/bin/bash
# v-tagged profile capture: launch list of prof_run C4 (3 reps) + full captures of the top kernels
V=$1
mkdir -p gpurun_out/prof_$V
if [ -z "$SKIP_LAUNCHES" ]; then
timeout 300 python tools/prof_run.py C4 3 > gpurun_out/prof_$V/plain.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/prof_$V/launches.csv python tools/prof_run.py C4 3 > gpurun_out/prof_$V/ncu_l.log 2>&1
fi
# skip the first rep's launches: the NB walk runs 6 times per call (build + rounds)
for ks in ${KERNELS:-k_walk<.int.0>:6 k_walk<.int.2>:1 k_force:1 k_density:1}; do
  k=${ks%%:*}; sk=${ks##*:}
  tag=$(echo $k | tr -d '<>.()' | sed 's/int//')
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:${k}" -s $sk -c 1 \
    -o gpurun_out/prof_$V/full_$tag python tools/prof_run.py C4 2 > gpurun_out/prof_$V/ncu_$tag.log 2>&1
done
ls -la gpurun_out/prof_$V
