cd /root/repo
for v in default old; do
  if [ $v != default ]; then export TXS_LIB=$PWD/build/var/libtxsite_$v.so; else unset TXS_LIB; fi
  TXS_VIX_DUAL=0 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:k_vix_lanes --csv --log-file gpurun_out/instcmp_$v.csv python profiles/scripts/stage_time.py c3 vix 1 > /dev/null 2>&1
  echo $v; grep -v "^==" gpurun_out/instcmp_$v.csv | awk -F'","' 'NR>1{print $5" | "$(NF-2)" "$NF}' | sed 's/(const short.*)//' | cut -c1-160
done
