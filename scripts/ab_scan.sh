# k_scan_emit duration per .so variant (ncu launch list of the headline step, 6 launches each)
cp paper_2412_13211_b200/libtrajlab_b200.so /tmp/orig.so
for m in ${VARIANTS:-base}; do
  cp scripts/_ab/$m.so paper_2412_13211_b200/libtrajlab_b200.so
  ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:k_scan_emit -s 2 -c 6 --csv python scripts/headline_step.py 8 2>/dev/null | grep k_scan_emit | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ' | sed "s/^/$m scan_emit ns (warm): /"; echo
done
cp /tmp/orig.so paper_2412_13211_b200/libtrajlab_b200.so
