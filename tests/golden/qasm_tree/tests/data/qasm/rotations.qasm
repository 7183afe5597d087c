OPENQASM 2.0;
include "qelib1.inc";
qreg q[2];
rx(pi/2) q[0];
ry(-pi/4) q[1];
rz(pi) q[0];
rz(2*pi/3) q[1];
