#!/bin/bash
# round-end evidence: GPU suite, smoke, bench (both arms), launch list + ncu --set full,
# the reference's own suite through the shim (needs .refcopy/ staged by the caller),
# bench lines of the other configs
cd "$(dirname "$0")/../.."
TAG=${TAG:-r2}
bash tools/jobs/r2_evidence.sh
if [ -d .refcopy/pkg ]; then
  (cd .refcopy && timeout 900 python ../tools/ref_suite/shim.py pkg pkg/tests -q -p no:cacheprovider -rA > ../gpurun_out/ref_suite_$TAG.log 2>&1; echo rc=$? >> ../gpurun_out/ref_suite_$TAG.log)
  tail -3 gpurun_out/ref_suite_$TAG.log
fi
bash tools/jobs/r2_configs.sh
