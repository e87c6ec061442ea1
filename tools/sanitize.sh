#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py
# (every launch layout), plus the hybrid cases through the global-memory slice
# paths (PK_FORCE_GLOBAL_SLICE=1|2).  Logs: $OUT/san_<tool>_<case>.log; one
# summary line per run on stdout.
OUT=${OUT:-gpurun_out/san}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
CASES=${CASES:-"cluster cluster128 packed sg single nv256 generic hybrid hybrid128 hybrid256 bigc bigw v3small chain parareal"}
TOOLS=${TOOLS:-"memcheck racecheck synccheck"}
for tool in $TOOLS; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  for c in $CASES; do
    for g in 0 1 2; do
      case "$c" in hybrid*) ;; *) [ "$g" != 0 ] && continue ;; esac
      tag="${tool}_${c}"; [ "$g" != 0 ] && tag="${tag}_global$g"
      if [ "$g" != 0 ]; then export PK_FORCE_GLOBAL_SLICE=$g; else unset PK_FORCE_GLOBAL_SLICE; fi
      timeout ${CASE_TIMEOUT:-900} $CS --tool $tool $extra --error-exitcode 3 \
        python tools/sanitize_cases.py --case $c > "$OUT/san_$tag.log" 2>&1
      rc=$?
      echo "$tag rc=$rc $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' "$OUT/san_$tag.log" | tr '\n' ' ')"
    done
  done
done
unset PK_FORCE_GLOBAL_SLICE
