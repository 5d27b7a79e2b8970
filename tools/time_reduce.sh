cd /root/repo
for sp in 0 1 2 3; do
  echo "splits=$sp: $(CPKIT_REDUCE_SPLITS=$sp ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:reduce python tools/profile_als.py 1 2>/dev/null | grep reduce | awk -F, '{print $(NF-0)}' | tr '\n' ' ')"
done
echo "generic: $(CPKIT_REDUCE_GENERIC=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:reduce python tools/profile_als.py 1 2>/dev/null | grep reduce | awk -F, '{print $(NF-0)}' | tr '\n' ' ')"
