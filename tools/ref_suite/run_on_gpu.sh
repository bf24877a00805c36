#!/usr/bin/env bash
# Run the reference's unmodified test suite on a B200 with the online path
# swapped for this package (tools/ref_suite/shim.py).  The reference copy is
# staged under .refcopy/ (git-ignored) only for the duration of the gpurun
# call: /root/reference does not exist on the GPU box.
set -euo pipefail
cd "$(dirname "$0")/../.."
rm -rf .refcopy && mkdir -p .refcopy && cp -r /root/reference/pkg .refcopy/pkg
trap 'rm -rf .refcopy' EXIT
/usr/local/graft/bin/gpurun --timeout "${TIMEOUT:-1200}" -- \
  "cd .refcopy && python ../tools/ref_suite/shim.py pkg pkg/tests -q -p no:cacheprovider -rA \
     > ../gpurun_out/ref_suite.log 2>&1; echo rc=\$? >> ../gpurun_out/ref_suite.log; \
   tail -5 ../gpurun_out/ref_suite.log"
