# ncu --set full of kernel $1 for every prebuilt abso/lib_*.so (copied over libws_b200.so)
for f in abso/lib_*.so; do
  n=$(basename $f .so)
  cp "$f" paper_2410_08946_b200/libws_b200.so
  bash tools/prof_one.sh "$1" 1 prof_${n}
done
