#!/usr/bin/env bash
# Regenerates the golden vectors from the REFERENCE implementation itself:
# oracle/_ref/ref_driver is built from /root/reference/proj/src by
# oracle/Makefile (reference flags, Eigen-subset shim). Run in the build
# container (needs /root/reference).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
make -s -C "$here/../../oracle" -j8
"$here/../../oracle/_ref/ref_driver" golden "$here" /root/reference/proj/data
gzip -f -9 "$here/instances_medium.json"
"$here/../../oracle/_ref/ref_driver" mantel_golden "$here"
"$here/../../oracle/_ref/ref_driver" wide_golden "$here"
gzip -f -9 "$here/instances_wide.json"
"$here/../../oracle/_ref/ref_driver" strf_golden "$here" /root/reference/proj/data
