run() { local name=$1; local cfg=$2; shift; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 "$cfg" > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2))")"; }
for i in 1 2 3; do
run cm10 '{}'
run cm105 '{}' SPH_COLD_MARGIN=1.05
run cm11 '{}' SPH_COLD_MARGIN=1.1
done
