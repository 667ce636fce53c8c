#!/bin/bash
# A/B of library builds on one workload: ab_syrk.sh W "label=path[:ENV=..]" ...
W=${W:-cfg3}
for spec in "$@"; do
  label=${spec%%=*}; rest=${spec#*=}; lib=${rest%%:*}; envs=""
  [[ "$rest" == *:* ]] && envs=${rest#*:}
  env E3_LIBCU=$lib $envs timeout 300 python tools/syrk_time.py --workload $W --tag "$label" ${ARGS:-} 2>&1 | tail -1
done
