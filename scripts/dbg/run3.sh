cd $(dirname $0)
for v in vA vB vD vE; do timeout 30 ./$v 31 31; done
