cd /root/repo
for shape in "400,400,400 100" "100,100,100,100 50" "200,200,200 20" "50,50,50 5" "200,200,200,200 200"; do
  echo "$shape: $(python tools/time_roots.py $shape 2>&1 | tail -1 | sed 's/dims=.*env=[^ ]* //')"
done
echo "C3 alt (7,1,3): $(CPKIT_TN_WM=7 CPKIT_TN_WN=1 CPKIT_TN_NTW=3 python tools/time_roots.py 200,200,200 20 2>&1 | tail -1 | sed 's/dims=.*env=[^ ]* //')"
