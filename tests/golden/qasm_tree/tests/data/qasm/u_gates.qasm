OPENQASM 2.0;
include "qelib1.inc";
qreg q[1];
u1(pi/8) q[0];
u2(0,pi) q[0];
u3(pi/2,-pi/2,pi/4) q[0];
