bash tools/full_quick.sh ${1:-fq}
bash tools/abso2.sh 2
