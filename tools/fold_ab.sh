# per-launch device time of the chunk fold for several builds (ncu launch list)
for v in "$@"; do
  SKV_LIB=ab/$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fold_rows --csv python tools/probe_text.py 2>/dev/null \
    | grep gpu__time | awk -F'","' -v t="$v" '{gsub(/"/,"",$NF); print t, $(NF-4), $NF}' | sed 's/(//;s/)//'
done
