run() { local name=$1; local cfg=$2; shift; shift; env "$@" timeout 300 python tools/prof_run.py C4 4 "$cfg" > gpurun_out/sw_$name.log 2>&1; echo "$name $(python -c "import json;d=json.loads(open('gpurun_out/sw_$name.log').read().strip().splitlines()[-1]);print(round(d['ms_build'],2),round(d['ms_density'],2),round(d['ms_force'],2),round(d['ms_total_events'],2))")"; }
run k1024 '{}'
run k1020 '{}' SPH_NBK=1020
run k1056 '{}' SPH_NBK=1056
run k996 '{}' SPH_NBK=996
run k516 '{}' SPH_NBK=516
run k1024b '{}'
