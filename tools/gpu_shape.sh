set -u
for args in "256 0" "240 0" "240 7" "256 7"; do timeout 60 ./tools/mxf4_probe pair $args; done
